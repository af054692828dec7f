#!/bin/bash
# compute-sanitizer over the global-state tier: state overflow,
# image overflow, u64 time range, explicit rows with out-of-range values
set -u
export PYTHONPATH=$PWD
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool global tier"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 5 python -m pytest -q -x tests/test_gpu_big.py \
      -k "tier_selection or (range_argmin and 4-wide) or (range_argmin and 2-long) or (explicit_rows and 3) or (u64 and 4)" 2>&1 | tail -5
done
