set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rs 2>&1 | tail -4 > gpurun_out/gpu_tests49.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke49.txt 2>&1
timeout 900 python bench.py --parity off --no-cpu-baseline > gpurun_out/bench49.json 2> gpurun_out/bench49.err
