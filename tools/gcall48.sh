set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rs 2>&1 | tail -8 > gpurun_out/gpu_tests48.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke48.txt 2>&1
