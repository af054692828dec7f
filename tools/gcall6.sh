set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_sym.py tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -5 > gpurun_out/gpu_tests6.txt
timeout 900 python tools/exact_bench.py > gpurun_out/exact6.jsonl 2> gpurun_out/exact6.err
timeout 1200 bash tools/np_ab_m.sh 4 > gpurun_out/np_ab_m4.txt 2>&1
timeout 1200 bash tools/np_ab_m.sh 8 > gpurun_out/np_ab_m8.txt 2>&1
