# NP A/B per workload at M = ${1:-4}: PP_NP pinned vs the rule vs PP_AUTOTUNE (10^9 placements/s)
M=${1:-4}
for w in gnmt biglstm inception_v3; do
 for np in "" 1 2 4 auto; do
  if [ "$np" = auto ]; then env_np="PP_AUTOTUNE=1"; else env_np="PP_NP=$np"; fi
  env $env_np PP_VERBOSE=1 timeout 300 python bench.py --workload $w --M $M --no-cpu-baseline --parity off --steps 3 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$w M=$M NP=${np:-rule}', round(d['value']/1e9,3), 'frac', round(d['roofline']['frac'],3))" 2>/dev/null || echo "$w NP=$np failed"
  grep "pp: M=$M" /tmp/b.err | tail -1
 done
done
