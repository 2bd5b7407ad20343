#!/bin/bash
# gpurun: K1 tests, then small-step / DCP timing for several K1 stream-K floors (DCP_K1_MIN_PAGES: an
# experiment build only -- the knob was not kept).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q -x tests/test_attention_gpu.py tests/test_dcp_step_gpu.py tests/test_step_graph_gpu.py tests/test_cfg1_gpu.py tests/test_cfg3_gpu.py > gpurun_out/pytest_k1min.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k1min.log
for M in 0 8 16 32 16 0; do
  echo "{\"min_pages\": $M}" >> gpurun_out/k1min.jsonl
  DCP_K1_MIN_PAGES=$M timeout 300 python bench_graph.py >> gpurun_out/k1min.jsonl 2>&1
  DCP_K1_MIN_PAGES=$M timeout 600 python bench_dcp.py --steps 150 >> gpurun_out/k1min.jsonl 2>> gpurun_out/k1min.err
done
DCP_K1_MIN_PAGES=16 timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-mla >> gpurun_out/k1min_bench.json 2>&1
