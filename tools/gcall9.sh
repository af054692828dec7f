set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -k "cut_words or perturb or fullsize or golden" 2>&1 | tail -3 > gpurun_out/gpu_tests9.txt
for w in inception_v3 gnmt biglstm; do
  echo "== $w M=4"; timeout 900 bash tools/ab_inception.sh --workload $w --M 4
done > gpurun_out/ab_mpw_prefetch.txt 2>&1
