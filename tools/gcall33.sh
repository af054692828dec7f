set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cold.py -m gpu -q -x 2>&1 | tail -25 > gpurun_out/gpu_cold33.txt
for M in 2 4 8; do for c in 0 1; do
  r=$(PP_COLD=$c PP_VERBOSE=1 timeout 600 python bench.py --workload gnmt --M $M --parity off --no-cpu-baseline --steps 3 --warmup 3 2> gpurun_out/cold33_err_${M}_${c}.txt | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,4), round(d['roofline']['frac'],4), d['result']['TM_ps'])")
  echo "gnmt M=$M PP_COLD=$c $r $(grep -m1 'pp: M=' gpurun_out/cold33_err_${M}_${c}.txt)"
done; done > gpurun_out/cold_ab33.txt 2>&1
