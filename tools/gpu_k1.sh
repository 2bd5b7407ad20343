#!/bin/bash
# gpurun: K1 parity (whole-frame + split rings, page sizes), racecheck of K1, bench.
set -u
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-k1}
timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_dcp_step_gpu.py tests/test_step_graph_gpu.py -m gpu -q > $OUT/pytest_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_$TAG.log
DCP_K1_SPLIT=1 timeout 900 python -m pytest tests/test_attention_gpu.py -m gpu -q > $OUT/pytest_split_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_split_$TAG.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest -q -m gpu -x \
   "tests/test_attention_gpu.py::test_small_shapes" "tests/test_attention_gpu.py::test_page_fill_non_final_partial" \
   "tests/test_attention_gpu.py::test_page_sizes" "tests/test_dcp_step_gpu.py" > $OUT/sanitize_racecheck_$TAG.log 2>&1; echo "exit=$?" >> $OUT/sanitize_racecheck_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
