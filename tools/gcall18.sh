set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_big.py -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests18.txt
for w in gnmt inception_v3; do for M in 2 4 8; do for c in 0 1; do
  r=$(PP_COLD=$c PP_VERBOSE=1 timeout 600 python bench.py --workload $w --M $M --parity off --no-cpu-baseline --steps 3 --warmup 3 2> gpurun_out/cold_err_${w}_${M}_${c}.txt | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,4), round(d['roofline']['frac'],4), d['result']['TM_ps'])")
  echo "$w M=$M PP_COLD=$c $r $(grep -m1 'pp: M=' gpurun_out/cold_err_${w}_${M}_${c}.txt)"
done; done; done > gpurun_out/cold_ab18.txt 2>&1
