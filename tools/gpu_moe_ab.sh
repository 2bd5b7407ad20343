#!/bin/bash
# gpurun: MoE tests + bench_moe (current build) and the routed DCP step tests.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest -m gpu -q -x tests/test_moe_gpu.py tests/test_cfg1_gpu.py > gpurun_out/pytest_moe_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_moe_ab.log
for r in 1 2; do timeout 300 python bench_moe.py >> gpurun_out/bench_moe_ab.jsonl 2>> gpurun_out/bench_moe_ab.err; done
