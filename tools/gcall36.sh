set -u
mkdir -p gpurun_out
timeout 1500 bash tools/np_ab_m.sh 4 > gpurun_out/np36_m4.txt 2>&1
timeout 1500 bash tools/np_ab_m.sh 8 > gpurun_out/np36_m8.txt 2>&1
timeout 1500 bash tools/np_ab_m.sh 2 > gpurun_out/np36_m2.txt 2>&1
