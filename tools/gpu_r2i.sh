#!/bin/bash
set -u
TAG=${1:-r2i}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_fused_step_gpu.py tests/test_layer_graph_gpu.py tests/test_multiproc_ipc_gpu.py tests/test_dcp_step_gpu.py tests/test_step_graph_gpu.py -m gpu -q -rA -s > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for a in "--reqs 16 --len 1000" "--reqs 4 --len 100" "--reqs 64 --len 2048"; do
  timeout 300 python tools/step_breakdown.py $a >> gpurun_out/breakdown_$TAG.jsonl 2>> gpurun_out/breakdown_$TAG.err
done
tail -3 gpurun_out/pytest_$TAG.log
