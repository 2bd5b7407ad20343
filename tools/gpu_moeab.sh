#!/bin/bash
# MoE A/B: bench_moe for the product build and each tools/probe/_bin/moe_* variant, twice, interleaved.
set -u
TAG=$1; shift
OUT=gpurun_out/moeab_$TAG
mkdir -p $OUT
L=paper_2605_21100_b200/_build/libdcp_b200.so
cp $L /tmp/lib_base.so
for rep in 1 2; do
for v in base "$@"; do
  if [ $v != base ]; then cp tools/probe/_bin/moe_$v/libdcp_b200.so $L; else cp /tmp/lib_base.so $L; fi
  timeout 300 python bench_moe.py --steps 30 > $OUT/bench_${v}_$rep.jsonl 2>&1
  if [ $rep = 1 ] && [ $v != base ]; then timeout 300 python -m pytest tests/test_moe_gpu.py tests/test_cfg1_gpu.py -m gpu -q -x > $OUT/pytest_$v.log 2>&1; echo "rc=$?" >> $OUT/pytest_$v.log; fi
done; done
cp /tmp/lib_base.so $L
