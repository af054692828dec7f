set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eft.py tests/test_gpu_fullsize.py tests/test_gpu_big.py -m gpu -q 2>&1 | tail -2 > gpurun_out/gpu_tests45.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke45.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches45.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --parity off > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches45.csv > gpurun_out/launches45_summary.txt 2>&1
timeout 900 python bench.py --parity off --no-cpu-baseline --steps 20 > gpurun_out/bench45.json 2> gpurun_out/bench45.err
