#!/bin/bash
# ncu --set full of one PERTURB search-kernel launch (Inception, M=2) for the
# default libpp.so and every tools/libpp_*.so variant; summaries to gpurun_out/
set -u
mkdir -p gpurun_out
cp paper_1907_13257_b200/libpp.so /tmp/libpp_default.so
for lib in /tmp/libpp_default.so tools/libpp_*.so; do
  [ -f "$lib" ] || continue
  n=$(basename $lib .so)
  cp "$lib" paper_1907_13257_b200/libpp.so
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:search_kernel -s 3 -c 1 \
    -o gpurun_out/ncu_$n -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_$n.ncu-rep > gpurun_out/ncu_$n.txt 2>&1
done
cp /tmp/libpp_default.so paper_1907_13257_b200/libpp.so
