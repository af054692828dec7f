set -u
mkdir -p gpurun_out
timeout 1500 bash tools/ab_inception.sh --parity off > gpurun_out/ab_ptxas34.txt 2>&1
