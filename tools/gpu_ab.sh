#!/bin/bash
# gpurun: K1 ring A/B — parity tests + bench for DCP_K1_SPLIT=0 and =1, ncu capture of the split variant.
set -u
TAG=${1:-ab}
OUT=gpurun_out; mkdir -p $OUT
DCP_K1_SPLIT=1 timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_dcp_step_gpu.py tests/test_step_graph_gpu.py -m gpu -q > $OUT/pytest_split_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_split_$TAG.log
for v in 0 1 0 1; do
  DCP_K1_SPLIT=$v timeout 300 python bench.py --no-cpu-baseline --steps 400 >> $OUT/bench_ab_$TAG.jsonl 2>> $OUT/bench_ab_$TAG.err
  echo "{\"variant\": $v}" >> $OUT/bench_ab_$TAG.jsonl
done
DCP_K1_SPLIT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:splitkv_decode -s 3 -c 1 \
    -o $OUT/k1split_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_split_$TAG.log 2>&1
echo done
