#!/bin/bash
# gpurun: compute-sanitizer over the kernels changed in round 2's last session (MoE single-release
# completion, warp-per-row K5b, fence-first / preloaded K4, K5c prefetch; the fused step's
# producer-side epoch ticket and 8-part K9 merge).
set -u
OUT=gpurun_out; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest -q -m gpu -x tests/test_moe_gpu.py tests/test_cfg1_gpu.py tests/test_fused_step_gpu.py \
      "tests/test_attention_gpu.py::test_cross_cta_splits" "tests/test_attention_gpu.py::test_tiny_grid_underfilled" "tests/test_attention_gpu.py::test_repeat_launch_counters_rearmed" > $OUT/sanitize6_$tool.log 2>&1
  echo "exit=$?" >> $OUT/sanitize6_$tool.log
done
