#!/bin/bash
# bench.py over workloads x M (PERTURB 10 x 1e7) — one line per case;
# extra arguments are passed to bench.py (e.g. --hw cube_mesh)
for w in inception_v3 gnmt biglstm; do
  for M in 2 4 8; do
    timeout 300 python bench.py --workload $w --M $M --no-cpu-baseline --steps 3 "$@" > /tmp/bm.json 2>/tmp/bm.err || { echo "$w M=$M failed"; tail -2 /tmp/bm.err; continue; }
    python -c "import json;d=json.load(open('/tmp/bm.json'));r=d['roofline'];print('$w M=$M', round(d['value']/1e9,3),'G/s frac',round(r['frac'],3),'SU',round(d['result']['su_mp'],4),'N*',d['result']['crossover_n_star'])"
  done
done
