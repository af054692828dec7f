#!/bin/bash
# compute-sanitizer over the smoke test and a small parity subset
set -u
export PYTHONPATH=$PWD
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool smoke"
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 5 python __graft_entry__.py 2>&1 | grep -E "ERROR SUMMARY|smoke ok|Error|error" | head -5
  echo "== $tool parity subset"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 5 python -m pytest -q -x tests/test_gpu_parity.py \
      -k "toy12_exhaustive or search_perturb_rounds and toy12 or memory_cap or every_placements_per_lane_variant and 1" 2>&1 | grep -E "ERROR SUMMARY|passed|failed|Error" | head -5
done
# round 2: the symmetry-reduced GRAY search (prefix reuse, NP = 3 at M = 3) and the
# M = 4, 8 device-word PERTURB schedule
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool sym + device words"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 5 python -m pytest -q -x tests/test_gpu_sym.py tests/test_gpu_parity.py \
      -k "(exhaustive_gray_equals_oracle and toy12 and (3 or 4)) or (cut_words and not memory_cap and 4-2)" 2>&1 | grep -E "ERROR SUMMARY|passed|failed|Error" | head -5
done
