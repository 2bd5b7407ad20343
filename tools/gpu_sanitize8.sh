#!/bin/bash
# gpurun: compute-sanitizer over the last round-2 changes: K1's per-shard routing fields (fused and
# routed steps), K10's PDL-chained launches (small MLA cases, graph replay, routed step).
set -u
OUT=gpurun_out; mkdir -p $OUT
T="tests/test_fused_step_gpu.py tests/test_dcp_step_gpu.py tests/test_mla_gpu.py::test_mla_edges tests/test_mla_gpu.py::test_mla_stream_k tests/test_mla_gpu.py::test_mla_graph_replay tests/test_mla_gpu.py::test_mla_routed_dcp_step"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest -q -m gpu -x $T > $OUT/sanitize8_$tool.log 2>&1
  echo "exit=$?" >> $OUT/sanitize8_$tool.log
done
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --error-exitcode 9 --print-limit 20 \
    python -m pytest -q -m gpu -x tests/test_multiproc_ipc_gpu.py > $OUT/sanitize8_memcheck_2proc.log 2>&1
echo "exit=$?" >> $OUT/sanitize8_memcheck_2proc.log
