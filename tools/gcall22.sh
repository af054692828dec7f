set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_big.py -m gpu -q 2>&1 | tail -5 > gpurun_out/gpu_big22.txt
