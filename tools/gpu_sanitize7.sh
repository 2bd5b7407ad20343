#!/bin/bash
# gpurun: compute-sanitizer over the end-of-round-2 changes: K10 with one P buffer and 4 + 4 PV
# stages (small MLA cases), the shared K5b/K5c bodies, and the fused MoE launches across two
# processes (--target-processes all).
set -u
OUT=gpurun_out; mkdir -p $OUT
MLA="tests/test_mla_gpu.py::test_mla_edges tests/test_mla_gpu.py::test_mla_stream_k tests/test_mla_gpu.py::test_mla_page_fill tests/test_mla_gpu.py::test_mla_routed_dcp_step"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest -q -m gpu -x $MLA tests/test_moe_gpu.py > $OUT/sanitize7_$tool.log 2>&1
  echo "exit=$?" >> $OUT/sanitize7_$tool.log
done
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --error-exitcode 9 --print-limit 20 \
    python -m pytest -q -m gpu -x tests/test_multiproc_ipc_gpu.py > $OUT/sanitize7_memcheck_2proc.log 2>&1
echo "exit=$?" >> $OUT/sanitize7_memcheck_2proc.log
