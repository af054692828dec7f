set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader > gpurun_out/box27.txt
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/gpu_tests27.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke27.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench27.json 2> gpurun_out/bench27.err
timeout 900 python bench.py --impl reference > gpurun_out/bench27_ref.json 2> gpurun_out/bench27_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_final27.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --parity off > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02_launches_final27.csv > gpurun_out/r02_launches_final27_summary.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/r02_ncu_m2_final27 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --parity off > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_ncu_m2_final27.ncu-rep > gpurun_out/r02_ncu_m2_final27.txt 2>&1
rm -f gpurun_out/*.ncu-rep
timeout 1200 bash tools/bench_matrix.sh > gpurun_out/matrix27.txt 2>&1
timeout 900 python tools/sweep.py --count 10000000 > gpurun_out/sweep27.jsonl 2> gpurun_out/sweep27.err
