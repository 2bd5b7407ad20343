#!/bin/bash
set -u
TAG=${1:-r2h}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_layer_graph_gpu.py tests/test_multiproc_ipc_gpu.py tests/test_moe_gpu.py -m gpu -q -rA -s > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench_moe.py --steps 20 > gpurun_out/bench_moe_$TAG.jsonl 2>&1
timeout 300 python bench_graph.py > gpurun_out/bench_graph_$TAG.json 2>&1
tail -3 gpurun_out/pytest_$TAG.log
