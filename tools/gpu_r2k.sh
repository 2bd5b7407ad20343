#!/bin/bash
set -u
TAG=${1:-r2k}
mkdir -p gpurun_out
timeout 300 python tools/k1_trace.py --sizes 4x100,16x1000 > gpurun_out/k1trace_local_$TAG.txt 2>&1
timeout 300 python tools/k1_trace.py --sizes 4x100,16x1000 --fused > gpurun_out/k1trace_fused_$TAG.txt 2>&1
timeout 900 python -m pytest tests/test_moe_gpu.py tests/test_layer_graph_gpu.py tests/test_fused_step_gpu.py -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench_moe.py --steps 20 > gpurun_out/bench_moe_$TAG.jsonl 2>&1
tail -2 gpurun_out/pytest_$TAG.log
