#!/bin/bash
# gpurun: compute-sanitizer memcheck / racecheck / synccheck over small parity cases of K1..K8.
set -u
OUT=gpurun_out; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest -q -m gpu -x \
      "tests/test_attention_gpu.py::test_small_shapes" \
      "tests/test_attention_gpu.py::test_cross_cta_splits" \
      "tests/test_planner_gpu.py::test_block_tables_match_page_table" \
      "tests/test_dcp_step_gpu.py" "tests/test_moe_gpu.py" \
      "tests/test_decode_growth_gpu.py::test_kv_append_writes_chosen_slot" \
      > $OUT/sanitize_$tool.log 2>&1
  echo "exit=$?" >> $OUT/sanitize_$tool.log
done
