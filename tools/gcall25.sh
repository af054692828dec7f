set -u
mkdir -p gpurun_out
timeout 1200 bash tools/bench_matrix.sh > gpurun_out/matrix25_rul10.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests25.txt
timeout 900 python tools/big_bench.py > gpurun_out/big_bench25.jsonl 2> gpurun_out/big_bench25.err
