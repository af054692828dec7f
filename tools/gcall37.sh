set -u
mkdir -p gpurun_out
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --parity off --no-cpu-baseline --steps 20 --warmup 3 > /tmp/b.json 2> /dev/null
  python -c "import json;d=json.load(open('/tmp/b.json'));print('run $i', round(d['value']/1e9,4), 'G/s frac', round(d['roofline']['frac'],4), 'kern_ms', round(d['roofline']['kernel_ms_avg'],4), 'e2e', round(d['e2e']['value']/1e9,4), 'clocks', d['clocks'])"
done > gpurun_out/bench_repeat37.txt 2>&1
