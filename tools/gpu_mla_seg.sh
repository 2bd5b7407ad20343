#!/bin/bash
# gpurun: K10 tests, then bench_mla for several stream-K shard-start weights (DCP_MLA_SEG_TILES).
set -u
TAG=${1:-seg}
mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q -x tests/test_mla_gpu.py > gpurun_out/pytest_mla_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mla_$TAG.log
for X in 0 4 8 12 16 8 0; do
  echo "{\"seg_tiles\": $X}" >> gpurun_out/bench_mla_$TAG.jsonl
  DCP_MLA_SEG_TILES=$X timeout 300 python bench_mla.py >> gpurun_out/bench_mla_$TAG.jsonl 2>> gpurun_out/bench_mla_$TAG.err
done
DCP_MLA_SEG_TILES=8 timeout 300 python tools/mla_trace.py > gpurun_out/mla_trace_$TAG.txt 2>&1
echo done
