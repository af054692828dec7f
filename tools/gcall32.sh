set -u
mkdir -p gpurun_out
timeout 1200 bash tools/ab_inception.sh --parity off > gpurun_out/ab_m2p32.txt 2>&1
