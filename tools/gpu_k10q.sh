#!/bin/bash
# gpurun: K10 tests + bench (QK chain balance), planner racecheck, planner tests.
set -u
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q -x tests/test_mla_gpu.py > gpurun_out/pytest_mla_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mla_$TAG.log
timeout 300 python bench_mla.py > gpurun_out/bench_mla_$TAG.jsonl 2> gpurun_out/bench_mla_$TAG.err
timeout 300 python tools/mla_trace.py > gpurun_out/mla_trace_$TAG.txt 2>&1
timeout 900 python -m pytest -m gpu -q -x tests/test_planner_gpu.py tests/test_decode_growth_gpu.py > gpurun_out/pytest_pl_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pl_$TAG.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest -q -m gpu -x \
   "tests/test_planner_gpu.py::test_block_tables_match_page_table" "tests/test_planner_gpu.py::test_routing_large_active_sets" \
   > gpurun_out/sanitize3_racecheck.log 2>&1; echo "exit=$?" >> gpurun_out/sanitize3_racecheck.log
echo done
