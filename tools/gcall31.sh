set -u
mkdir -p gpurun_out
timeout 900 bash tools/ab_inception.sh --parity off --workload gnmt --M 4 > gpurun_out/ab_extra31.txt 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --M 4 >> gpurun_out/ab_extra31.txt 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --workload gnmt --M 8 >> gpurun_out/ab_extra31.txt 2>&1
