#!/bin/bash
set -u
TAG=${1:-r2l}
mkdir -p gpurun_out
bash tools/gpu_k1iter.sh $TAG
DCP_K1_MERGE=last timeout 300 python tools/probe_k1_small.py > gpurun_out/k1small_last_$TAG.jsonl 2>&1
timeout 300 python tools/k1_trace.py --sizes 4x100,16x1000 --fused > gpurun_out/k1trace_fused_$TAG.txt 2>&1
timeout 900 python -m pytest tests/test_fused_step_gpu.py tests/test_multiproc_ipc_gpu.py tests/test_layer_graph_gpu.py -m gpu -q -x > gpurun_out/pytest2_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest2_$TAG.log
tail -2 gpurun_out/pytest2_$TAG.log
