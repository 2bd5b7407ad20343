#!/bin/bash
set -u
TAG=${1:-r2g}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_layer_graph_gpu.py tests/test_moe_gpu.py tests/test_step_graph_gpu.py -m gpu -q -rA -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
bash tools/gpu_k1iter.sh ${TAG}k1
tail -3 gpurun_out/pytest_$TAG.log
