#!/bin/bash
# build_variant.sh NAME "NVCC FLAGS": builds libpp.so with extra nvcc flags
# into tools/libpp_NAME.so (A/B experiments), leaving the default build in place
set -eu
cp paper_1907_13257_b200/libpp.so /tmp/libpp_keep.so
PP_NVCC_FLAGS="$2" python -c "from paper_1907_13257_b200 import _build; _build.build(force=True)"
cp paper_1907_13257_b200/libpp.so tools/libpp_$1.so
cp /tmp/libpp_keep.so paper_1907_13257_b200/libpp.so
touch paper_1907_13257_b200/libpp.so
