set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests13.txt
timeout 900 python -m pytest tests/test_gpu_big.py -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_big13.txt
timeout 900 python bench.py --parity off --no-cpu-baseline > gpurun_out/bench13.json 2> gpurun_out/bench13.err
timeout 1500 bash tools/sanitize_big.sh > gpurun_out/sanitize_big13.txt 2>&1
