set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests46.txt
timeout 900 python bench.py > gpurun_out/bench46.json 2> gpurun_out/bench46.err
