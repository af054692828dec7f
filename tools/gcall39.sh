set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_big.py -m gpu -q 2>&1 | tail -2 > gpurun_out/gpu_big39.txt
timeout 900 python tools/big_bench.py > gpurun_out/big_bench39.jsonl 2> gpurun_out/big_bench39.err
