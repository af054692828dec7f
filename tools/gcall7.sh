set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests7.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke7.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err
timeout 900 python bench.py --impl reference > gpurun_out/bench7_ref.json 2> gpurun_out/bench7_ref.err
timeout 900 bash tools/bench_matrix.sh > gpurun_out/matrix7.txt 2>&1
timeout 900 python tools/exact_bench.py > gpurun_out/exact7.jsonl 2> gpurun_out/exact7.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/r02_ncu_gnmt_m4 -f python bench.py --workload gnmt --M 4 --steps 1 --warmup 0 --no-cpu-baseline --parity off > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel -s 3 -c 1 \
  -o gpurun_out/r02_ncu_m4v17 -f python bench.py --M 4 --steps 1 --warmup 0 --no-cpu-baseline --parity off > /dev/null 2>&1
for f in r02_ncu_gnmt_m4 r02_ncu_m4v17; do python tools/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/$f.txt 2>&1; done
rm -f gpurun_out/*.ncu-rep
