set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/gpu_tests5.txt
timeout 600 python tools/sym_bench.py > gpurun_out/sym_bench5.jsonl 2> gpurun_out/sym_bench5.err
timeout 900 python bench.py > gpurun_out/bench5.json 2> gpurun_out/bench5.err
timeout 900 bash tools/bench_matrix.sh > gpurun_out/matrix5.txt 2>&1
timeout 900 python tools/sweep.py --count 10000000 > gpurun_out/sweep5.jsonl 2> gpurun_out/sweep5.err
timeout 900 python tools/exact_bench.py > gpurun_out/exact5.jsonl 2> gpurun_out/exact5.err
timeout 2400 bash tools/sanitize.sh > gpurun_out/sanitize5.txt 2>&1
