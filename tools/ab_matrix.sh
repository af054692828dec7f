#!/bin/bash
# A/B over alternative libpp.so builds (tools/libpp_*.so): bench_matrix per build
set -u
cp paper_1907_13257_b200/libpp.so /tmp/libpp_default.so
for lib in /tmp/libpp_default.so tools/libpp_*.so; do
  [ -f "$lib" ] || continue
  echo "### $(basename $lib)"
  cp "$lib" paper_1907_13257_b200/libpp.so
  bash tools/bench_matrix.sh "$@"
done
cp /tmp/libpp_default.so paper_1907_13257_b200/libpp.so
