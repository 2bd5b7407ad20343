#!/bin/bash
# gpurun: compute-sanitizer over the MoE (K4/K5) and K7 routing kernels changed at the end of round 1.
set -u
OUT=gpurun_out; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest -q -m gpu -x "tests/test_moe_gpu.py" "tests/test_cfg1_gpu.py" \
      "tests/test_planner_gpu.py::test_routing_large_active_sets" "tests/test_planner_gpu.py::test_block_tables_match_page_table" \
      > $OUT/sanitize3_$tool.log 2>&1
  echo "exit=$?" >> $OUT/sanitize3_$tool.log
done
