set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_big.py -m gpu -q 2>&1 | tail -15 > gpurun_out/gpu_big11.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests11.txt
timeout 900 python tools/big_bench.py > gpurun_out/big_bench11.jsonl 2> gpurun_out/big_bench11.err
