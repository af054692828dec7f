#!/bin/bash
# A/B: Inception M=2 PERTURB, 3 runs per libpp build (tools/libpp_*.so vs the in-tree build)
cp paper_1907_13257_b200/libpp.so /tmp/libpp_default.so
for rep in 1 2 3; do
  for lib in /tmp/libpp_default.so tools/libpp_*.so; do
    cp "$lib" paper_1907_13257_b200/libpp.so
    timeout 300 python bench.py --no-cpu-baseline --steps 5 "$@" > /tmp/ab.json 2>/dev/null
    python -c "import json;d=json.load(open('/tmp/ab.json'));print('$(basename $lib)', round(d['value']/1e9,4), 'kern_ms', round(d['roofline']['kernel_ms_avg'],4))"
  done
done
cp /tmp/libpp_default.so paper_1907_13257_b200/libpp.so
