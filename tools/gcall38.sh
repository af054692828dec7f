set -u
mkdir -p gpurun_out
cp paper_1907_13257_b200/libpp.so /tmp/libpp_default.so
timeout 900 python -m pytest tests/test_gpu_big.py -m gpu -q 2>&1 | tail -2 > gpurun_out/gpu_big38.txt
for lib in /tmp/libpp_default.so tools/libpp_pf0m2.so tools/libpp_pf0m4.so; do
  cp $lib paper_1907_13257_b200/libpp.so
  echo "== $(basename $lib)"
  timeout 900 python tools/big_bench.py 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l)
    if d['tier']=='global' and d['state_mb'] in ('4096',): print(d['dfg'], d['M'], '%.4g'%d['placements_per_s'], round(d['frac'],4))"
done > gpurun_out/big_pf38.txt 2>&1
cp /tmp/libpp_default.so paper_1907_13257_b200/libpp.so
