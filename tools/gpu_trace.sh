#!/bin/bash
# gpurun: trace-driven serving bench — the default run plus P99-TPOT rate sweeps (1% and 5% long).
set -u
TAG=${1:-tr}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python bench_trace.py --rate 16 > $OUT/bench_trace_$TAG.jsonl 2> $OUT/bench_trace_$TAG.err
for LR in 0.05 0.01; do
  timeout 2400 python bench_trace.py --sweep-rates 16,32,48,64,96,128 --long-ratio $LR --duration 10 --slo-ms 20 \
      > $OUT/bench_trace_sweep${LR}_$TAG.jsonl 2> $OUT/bench_trace_sweep${LR}_$TAG.err
done
echo done
