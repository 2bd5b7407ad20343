#!/bin/bash
set -u
TAG=${1:-r2o}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_planner_gpu.py tests/test_dropin_gpu.py tests/test_layer_graph_gpu.py tests/test_step_graph_gpu.py -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-mla > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/pytest_$TAG.log
