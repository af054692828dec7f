set -u
mkdir -p gpurun_out
timeout 900 bash tools/ab_inception.sh --parity off --M 4 > gpurun_out/ab_recpf40.txt 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --M 4 --workload gnmt >> gpurun_out/ab_recpf40.txt 2>&1
timeout 900 bash tools/ab_inception.sh --parity off --M 4 --workload biglstm >> gpurun_out/ab_recpf40.txt 2>&1
