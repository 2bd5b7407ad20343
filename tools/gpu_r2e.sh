#!/bin/bash
set -u
TAG=${1:-r2e}
mkdir -p gpurun_out
timeout 300 python tools/k1_trace.py > gpurun_out/k1trace_$TAG.txt 2>&1
timeout 900 python -m pytest tests/test_kv_migrate_gpu.py -m gpu -q -rA -s > gpurun_out/pytest_$TAG.log 2>&1
echo done
