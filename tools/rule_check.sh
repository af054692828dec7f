bash tools/bench_matrix.sh 2>&1 | sed 's/^/rule /'
PP_AUTOTUNE=1 bash tools/bench_matrix.sh 2>&1 | sed 's/^/auto /'
for w in inception_v3 gnmt biglstm; do for M in 2 4 8; do PP_VERBOSE=1 timeout 120 python bench.py --workload $w --M $M --no-cpu-baseline --steps 1 --warmup 1 --rounds 1 2>&1 >/dev/null | grep "pp: M" | sort -u | head -1 | sed "s/^/$w /"; done; done
python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print('value', d['value'], 'e2e', d['e2e']['value'])"
