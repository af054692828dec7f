# Everything the round's profiles come from, on one B200 box (gpurun):
#   bash tools/round_check.sh   -> gpurun_out/
# (compute-sanitizer is closed on the GPU pool since round 2; tools/sanitize.sh
#  is kept for boxes where it is allowed)
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader > gpurun_out/box.txt
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --parity off > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_m2 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --parity off > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu_m2.ncu-rep > gpurun_out/ncu_m2.txt 2>&1
rm -f gpurun_out/*.ncu-rep
timeout 1200 bash tools/bench_matrix.sh > gpurun_out/matrix.txt 2>&1
timeout 900 python tools/sweep.py --count 10000000 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 900 python tools/exact_bench.py > gpurun_out/exact.jsonl 2> gpurun_out/exact.err
timeout 900 python tools/sym_bench.py > gpurun_out/sym_bench.jsonl 2> gpurun_out/sym_bench.err
timeout 900 python tools/pipeline_bench.py > gpurun_out/pipeline.jsonl 2> gpurun_out/pipeline.err
timeout 900 python tools/big_bench.py > gpurun_out/big_bench.jsonl 2> gpurun_out/big_bench.err
