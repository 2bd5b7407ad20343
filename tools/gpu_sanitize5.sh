#!/bin/bash
# gpurun: memcheck over the K10 (MLA), K1 attention, routed-step and step-graph suites.
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
    python -m pytest -q -m gpu -x tests/test_mla_gpu.py tests/test_attention_gpu.py tests/test_dcp_step_gpu.py \
    tests/test_step_graph_gpu.py > $OUT/sanitize5_memcheck.log 2>&1
echo "exit=$?" >> $OUT/sanitize5_memcheck.log
