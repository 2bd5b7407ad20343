#!/bin/bash
# gpurun: compute-sanitizer over the planner / routing / K10 paths changed late in round 1.
set -u
OUT=gpurun_out; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest -q -m gpu -x \
      "tests/test_planner_gpu.py::test_block_tables_match_page_table" \
      "tests/test_planner_gpu.py::test_routing_large_active_sets" \
      "tests/test_planner_gpu.py::test_golden_scenarios" \
      "tests/test_decode_growth_gpu.py" \
      > $OUT/sanitize2_$tool.log 2>&1
  echo "exit=$?" >> $OUT/sanitize2_$tool.log
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
    python -m pytest -q -m gpu -x "tests/test_mla_gpu.py::test_mla_edges" > $OUT/sanitize2_mla_memcheck.log 2>&1
echo "exit=$?" >> $OUT/sanitize2_mla_memcheck.log
