set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests43.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke43.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench43.json 2> gpurun_out/bench43.err
timeout 900 python bench.py --impl reference > gpurun_out/bench43_ref.json 2> gpurun_out/bench43_ref.err
timeout 1200 bash tools/bench_matrix.sh > gpurun_out/matrix43.txt 2>&1
timeout 900 python tools/sweep.py --count 10000000 > gpurun_out/sweep43.jsonl 2> gpurun_out/sweep43.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches43.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --parity off > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches43.csv > gpurun_out/launches43_summary.txt 2>&1
