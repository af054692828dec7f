set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "cut_words or perturb or toy12" 2>&1 | tail -2 > gpurun_out/gpu_tests44.txt
timeout 900 bash tools/ab_inception.sh --parity off > gpurun_out/ab_bw44.txt 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --workload gnmt >> gpurun_out/ab_bw44.txt 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --workload biglstm >> gpurun_out/ab_bw44.txt 2>&1
