#!/bin/bash
# bench_matrix (workloads x M, PERTURB) + RANDOM M=2/4 for the default libpp.so
# and every tools/libpp_*.so variant
set -u
cp paper_1907_13257_b200/libpp.so /tmp/libpp_default.so
for lib in /tmp/libpp_default.so tools/libpp_*.so; do
  [ -f "$lib" ] || continue
  cp "$lib" paper_1907_13257_b200/libpp.so
  echo "== $(basename $lib)"
  bash tools/bench_matrix.sh
  for M in 2 4; do
    timeout 300 python bench.py --gen random --count 100000000 --M $M --no-cpu-baseline --steps 3 > /tmp/bm.json 2>/dev/null
    python -c "import json;d=json.load(open('/tmp/bm.json'));print('inception RANDOM M=$M', round(d['value']/1e9,3),'G/s frac',round(d['roofline']['frac'],3))"
  done
done
cp /tmp/libpp_default.so paper_1907_13257_b200/libpp.so
