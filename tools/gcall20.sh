set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader > gpurun_out/box20.txt
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/gpu_tests20.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke20.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench20.json 2> gpurun_out/bench20.err
timeout 900 python bench.py --impl reference > gpurun_out/bench20_ref.json 2> gpurun_out/bench20_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_final.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --parity off > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02_launches_final.csv > gpurun_out/r02_launches_final_summary.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/r02_ncu_m2_final -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --parity off > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_ncu_m2_final.ncu-rep > gpurun_out/r02_ncu_m2_final.txt 2>&1
rm -f gpurun_out/*.ncu-rep
timeout 1200 bash tools/bench_matrix.sh > gpurun_out/matrix20.txt 2>&1
timeout 900 python tools/sweep.py --count 10000000 > gpurun_out/sweep20.jsonl 2> gpurun_out/sweep20.err
