#!/bin/bash
# gpurun: K1 iteration check — K1/routed/cfg tests, per-CTA trace, small-batch probe, step breakdown, bench.
#   bash tools/gpu_k1iter.sh TAG
set -u
TAG=${1:-k1it}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_attention_gpu.py tests/test_dcp_step_gpu.py tests/test_cfg1_gpu.py \
    tests/test_cfg3_gpu.py tests/test_decode_growth_gpu.py tests/test_step_graph_gpu.py tests/test_kv_migrate_gpu.py \
    tests/test_multiproc_ipc_gpu.py tests/test_exchange_protocol_gpu.py -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python tools/k1_trace.py > gpurun_out/k1trace_$TAG.txt 2>&1
timeout 300 python tools/probe_k1_small.py > gpurun_out/k1small_$TAG.jsonl 2>&1
for a in "--reqs 16 --len 1000" "--reqs 64 --len 2048" "--reqs 4 --len 100"; do
  timeout 300 python tools/step_breakdown.py $a >> gpurun_out/breakdown_$TAG.jsonl 2>> gpurun_out/breakdown_$TAG.err
done
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-mla > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/pytest_$TAG.log
