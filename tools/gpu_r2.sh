#!/bin/bash
# gpurun: round-2 check — GPU tests (+durations), smoke, MoE bench.  bash tools/gpu_r2.sh TAG [pytest-args]
set -u
TAG=${1:-r2}
shift || true
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=15 "$@" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 300 python bench_moe.py --steps 20 > gpurun_out/bench_moe_$TAG.jsonl 2>&1; echo "moe rc=$?" >> gpurun_out/bench_moe_$TAG.jsonl
tail -5 gpurun_out/pytest_gpu_$TAG.log
