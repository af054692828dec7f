set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/gpu_tests3.txt
timeout 600 python tools/sym_bench.py > gpurun_out/sym_bench3.jsonl 2> gpurun_out/sym_bench3.err
timeout 900 python tools/local_opt.py > gpurun_out/local_opt.jsonl 2> gpurun_out/local_opt.err
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err
timeout 900 bash tools/ab_inception.sh > gpurun_out/ab_mix.txt 2>&1
timeout 900 bash tools/bench_matrix.sh > gpurun_out/matrix3.txt 2>&1
