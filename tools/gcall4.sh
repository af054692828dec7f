set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/gpu_tests4.txt
timeout 600 python tools/sym_bench.py > gpurun_out/sym_bench4.jsonl 2> gpurun_out/sym_bench4.err
# launch list of the default bench (per-launch durations, cold and serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --parity off > /dev/null 2>&1
# full capture of one headline search-kernel launch (Inception M=2 PERTURB) and of M=4 (device words)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/r02_ncu_m2 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --parity off > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/r02_ncu_m4 -f python bench.py --M 4 --steps 1 --warmup 0 --no-cpu-baseline --parity off > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/r02_ncu_gnmt_m2 -f python bench.py --workload gnmt --steps 1 --warmup 0 --no-cpu-baseline --parity off > /dev/null 2>&1
for f in r02_ncu_m2 r02_ncu_m4 r02_ncu_gnmt_m2; do python tools/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/$f.txt 2>&1; done
rm -f gpurun_out/*.ncu-rep
