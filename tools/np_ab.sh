for w in gnmt biglstm inception_v3; do
 for np in "" 1 2 4; do
  PP_NP=$np PP_VERBOSE=1 timeout 300 python bench.py --workload $w --M 2 --no-cpu-baseline --steps 3 > /tmp/b.json 2>/tmp/b.err
  python -c "import json;d=json.load(open('/tmp/b.json'));print('$w NP=${np:-rule}', round(d['value']/1e9,3))" 2>/dev/null || echo "$w NP=$np failed"
  grep "pp: M=2" /tmp/b.err | head -1
 done
done
