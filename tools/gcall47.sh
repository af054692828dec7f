set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sym.py -m gpu -q -rs 2>&1 | tail -8 > gpurun_out/gpu_sym47.txt
