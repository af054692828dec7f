set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q 2>&1 | tail -2 > gpurun_out/gpu_tests42.txt
for w in gnmt inception_v3 biglstm; do for rp in 0 1; do
  r=$(PP_RP=$rp PP_VERBOSE=1 timeout 600 python bench.py --workload $w --M 2 --parity off --no-cpu-baseline --steps 3 --warmup 3 2> gpurun_out/rp42_err.txt | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,4), round(d['roofline']['frac'],4))")
  echo "$w M=2 PP_RP=$rp $r $(grep -m1 'pp: M=' gpurun_out/rp42_err.txt)"
done; done > gpurun_out/rp_ab42.txt 2>&1
