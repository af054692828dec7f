set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests35.txt
timeout 900 bash tools/ab_inception.sh --parity off --M 4 > gpurun_out/ab_lazy35.txt 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --M 4 --workload gnmt >> gpurun_out/ab_lazy35.txt 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --M 4 --workload biglstm >> gpurun_out/ab_lazy35.txt 2>&1
