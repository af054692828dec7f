set -u
mkdir -p gpurun_out
timeout 900 python tools/pipeline_bench.py > gpurun_out/pipeline16.jsonl 2> gpurun_out/pipeline16.err
for c in wide long; do
  timeout 900 python tools/big_one.py $c > gpurun_out/big_one_$c.txt 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_big_kernel -s 2 -c 1 \
    -o gpurun_out/r02_ncu_big_$c -f python tools/big_one.py $c > gpurun_out/ncu_big_$c.log 2>&1
  python tools/ncu_summary.py gpurun_out/r02_ncu_big_$c.ncu-rep > gpurun_out/r02_ncu_big_$c.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
