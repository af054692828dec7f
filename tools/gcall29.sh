set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests29.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke29.txt 2>&1
timeout 1200 bash tools/bench_matrix.sh > gpurun_out/matrix29.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench29.json 2> gpurun_out/bench29.err
