#!/bin/bash
set -u
TAG=${1:-r2m}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_moe_gpu.py tests/test_fused_step_gpu.py tests/test_dcp_step_gpu.py tests/test_layer_graph_gpu.py tests/test_multiproc_ipc_gpu.py tests/test_planner_gpu.py -m gpu -q -rA -s > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for a in "--reqs 16 --len 1000" "--reqs 4 --len 100"; do
  timeout 300 python tools/step_breakdown.py $a >> gpurun_out/breakdown_$TAG.jsonl 2>> gpurun_out/breakdown_$TAG.err
done
timeout 900 python bench_trace.py --duration 5 --rate 16 --policies dcp,least_cache > gpurun_out/bench_trace_$TAG.jsonl 2> gpurun_out/bench_trace_$TAG.err
tail -3 gpurun_out/pytest_$TAG.log
