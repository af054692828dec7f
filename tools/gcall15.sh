set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sym.py tests/test_gpu_exact.py tests/test_gpu_pipeline.py tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -4 > gpurun_out/gpu_tests15.txt
timeout 900 python tools/sym_bench.py > gpurun_out/sym_bench15.jsonl 2> gpurun_out/sym_bench15.err
timeout 900 python tools/exact_bench.py > gpurun_out/exact15.jsonl 2> gpurun_out/exact15.err
timeout 900 python tools/pipeline_bench.py > gpurun_out/pipeline15.jsonl 2> gpurun_out/pipeline15.err
