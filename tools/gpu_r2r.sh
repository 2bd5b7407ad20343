#!/bin/bash
# r2r: MMA shape probe; K6 PDL-trigger fix; K6 CP-1 batch A/B
set -u
mkdir -p gpurun_out
timeout 120 tools/probe/_bin/mma_shape > gpurun_out/mma_shape.txt 2>&1
for r in 1 2 3; do timeout 300 python tools/planner_prof.py >> gpurun_out/k6_batch.txt 2>&1; done
cp paper_2605_21100_b200/_build/libdcp_b200.so /tmp/lib_default.so
cp tools/probe/_bin/nob/libdcp_b200.so paper_2605_21100_b200/_build/libdcp_b200.so
for r in 1 2 3; do timeout 300 python tools/planner_prof.py >> gpurun_out/k6_nobatch.txt 2>&1; done
cp /tmp/lib_default.so paper_2605_21100_b200/_build/libdcp_b200.so
timeout 600 python -m pytest tests/test_planner_gpu.py tests/test_dropin_gpu.py -m gpu -q -x > gpurun_out/pytest_r2r.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r2r.log
