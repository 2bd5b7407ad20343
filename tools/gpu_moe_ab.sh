#!/bin/bash
# gpurun: MoE tests + bench_moe for several chunk counts (DCP_MOE_CHUNKS).
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest -m gpu -q -x tests/test_moe_gpu.py > gpurun_out/pytest_moe_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_moe_ab.log
for C in 32 64 128 32 128; do
  echo "{\"chunks\": $C}" >> gpurun_out/bench_moe_ab.jsonl
  DCP_MOE_CHUNKS=$C timeout 300 python bench_moe.py >> gpurun_out/bench_moe_ab.jsonl 2>> gpurun_out/bench_moe_ab.err
done
DCP_MOE_CHUNKS=128 timeout 600 python -m pytest -m gpu -q -x tests/test_moe_gpu.py > gpurun_out/pytest_moe_ab128.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_moe_ab128.log
