#!/bin/bash
set -u
TAG=${1:-moe2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_moe_gpu.py tests/test_cfg1_gpu.py tests/test_multiproc_ipc_gpu.py tests/test_layer_graph_gpu.py tests/test_exchange_protocol_gpu.py tests/test_fused_step_gpu.py -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench_moe.py --steps 30 > gpurun_out/bench_moe_$TAG.jsonl 2>&1
