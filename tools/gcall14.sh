set -u
mkdir -p gpurun_out
timeout 900 python tools/sym_bench.py > gpurun_out/sym_bench14.jsonl 2> gpurun_out/sym_bench14.err
timeout 1500 bash tools/sanitize_big.sh > gpurun_out/sanitize_big14.txt 2>&1
