#!/bin/bash
# A/B: bench PERTURB and RANDOM with alternative libpp.so builds (tools/libpp_*.so,
# tools/build_variant.sh); each variant also runs the M = 2 PERTURB parity test
set -u
cp paper_1907_13257_b200/libpp.so /tmp/libpp_default.so
for lib in /tmp/libpp_default.so tools/libpp_*.so; do
  [ -f "$lib" ] || continue
  cp "$lib" paper_1907_13257_b200/libpp.so
  par=$(timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "cut_words or perturb_rounds" 2>&1 | tail -1)
  for g in perturb random; do
    c=$([ $g = random ] && echo 100000000 || echo 10000000)
    timeout 300 python bench.py --gen $g --count $c --no-cpu-baseline --steps 3 > /tmp/ab.json 2>/dev/null
    python -c "import json,sys;d=json.load(open('/tmp/ab.json'));print('$(basename $lib) $g', round(d['value']/1e9,3), 'G/s frac', round(d['roofline']['frac'],3), 'kern_ms', round(d['roofline']['kernel_ms_avg'],3))"
  done
  echo "   parity: $par"
done
cp /tmp/libpp_default.so paper_1907_13257_b200/libpp.so
