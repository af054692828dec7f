set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader > gpurun_out/box.txt
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gpu_tests.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
bash tools/bench_matrix.sh > gpurun_out/matrix.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_pipes tools/mb_pipes.cu && /tmp/mb_pipes > gpurun_out/mb_pipes.txt 2>&1
