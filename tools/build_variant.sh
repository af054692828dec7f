#!/bin/bash
# build_variant.sh NAME "NVCC FLAGS" [M]: relinks libpp.so with search_m<M>.o (the
# kernels of device count M, default 2) recompiled with extra nvcc flags, into
# tools/libpp_NAME.so (A/B experiments); the default build in paper_1907_13257_b200/
# is untouched
set -eu
M=${3:-2}
B=paper_1907_13257_b200/build
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I include -Xptxas --register-usage-level=10 $2 -DPP_M=$M \
  -c paper_1907_13257_b200/csrc/search_inst.cu -o /tmp/search_m${M}_$1.o 2>/dev/null
objs=""
for o in search_m1 search_m2 search_m3 search_m4 search_m5 search_m6 search_m7 search_m8 projection eft pipeline loader capi; do
  if [ $o = search_m$M ]; then objs="$objs /tmp/search_m${M}_$1.o"; else objs="$objs $B/$o.o"; fi
done
nvcc $ARCH -shared -o tools/libpp_$1.so $objs -ldl
