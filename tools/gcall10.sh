set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader > gpurun_out/box10.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests10.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke10.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench10.json 2> gpurun_out/bench10.err
