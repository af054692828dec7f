set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "not fullsize" 2>&1 | tail -30 > gpurun_out/gpu_tests2.txt
timeout 600 python tools/sym_bench.py > gpurun_out/sym_bench.jsonl 2> gpurun_out/sym_bench.err
timeout 900 python tools/tau_scan.py > gpurun_out/tau_scan.jsonl 2> gpurun_out/tau_scan.err
timeout 900 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err
