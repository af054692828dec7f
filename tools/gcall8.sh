set -u
mkdir -p gpurun_out
timeout 900 bash tools/ab_inception.sh > gpurun_out/ab_tiles_inception.txt 2>&1
timeout 900 bash tools/ab_inception.sh --workload gnmt > gpurun_out/ab_tiles_gnmt.txt 2>&1
timeout 900 bash tools/ab_inception.sh --workload biglstm > gpurun_out/ab_tiles_biglstm.txt 2>&1
