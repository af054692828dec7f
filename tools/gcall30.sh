set -u
mkdir -p gpurun_out
timeout 900 bash tools/ab_inception.sh --parity off > gpurun_out/ab_extra30.txt 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --workload gnmt >> gpurun_out/ab_extra30.txt 2>&1
rm -f tools/libpp_*.so
bash tools/build_variant.sh xs0m4 "-DPP_EXTRA_SPLIT=0" 4 > /dev/null 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --workload gnmt --M 4 >> gpurun_out/ab_extra30.txt 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --M 4 >> gpurun_out/ab_extra30.txt 2>&1
