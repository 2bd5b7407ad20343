#!/bin/bash
# gpurun: planner parity tests + the bench.py planner scenario (new build, then an optional A/B build).
set -u
TAG=${1:-pl}
AB=${2:-}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest -m gpu -q -x tests/test_planner_gpu.py tests/test_dropin_gpu.py tests/test_decode_growth_gpu.py tests/test_dcp_step_gpu.py > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_$TAG.log
for r in 1 2 3; do timeout 300 python tools/planner_prof.py >> $OUT/planner_$TAG.txt 2>&1; done
if [ -n "$AB" ]; then
  cp $AB/libdcp_b200.so paper_2605_21100_b200/_build/libdcp_b200.so
  for r in 1 2 3; do timeout 300 python tools/planner_prof.py >> $OUT/planner_${TAG}_ab.txt 2>&1; done
fi
echo done
