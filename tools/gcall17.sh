set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests17.txt
timeout 900 python tools/big_bench.py > gpurun_out/big_bench17.jsonl 2> gpurun_out/big_bench17.err
timeout 900 python tools/pipeline_bench.py > gpurun_out/pipeline17.jsonl 2> gpurun_out/pipeline17.err
timeout 900 python bench.py --parity off --no-cpu-baseline > gpurun_out/bench17.json 2> gpurun_out/bench17.err
for c in long; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_big_kernel -s 2 -c 1 \
    -o gpurun_out/r02_ncu_big_f64_$c -f python tools/big_one.py $c > gpurun_out/ncu_big_f64_$c.log 2>&1
  python tools/ncu_summary.py gpurun_out/r02_ncu_big_f64_$c.ncu-rep > gpurun_out/r02_ncu_big_f64_$c.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
