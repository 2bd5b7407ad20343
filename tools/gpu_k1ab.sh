#!/bin/bash
# K1 small-step A/B: step_breakdown (16x1000, 4x100) + k1 traces for the product build and each
# tools/probe/_bin/<variant>; K1 / fused-step parity tests for each variant.
set -u
TAG=$1; shift
OUT=gpurun_out/k1ab_$TAG
mkdir -p $OUT
L=paper_2605_21100_b200/_build/libdcp_b200.so
cp $L /tmp/lib_base.so
for rep in 1 2; do
for v in base "$@"; do
  if [ $v != base ]; then cp tools/probe/_bin/$v/libdcp_b200.so $L; else cp /tmp/lib_base.so $L; fi
  timeout 200 python tools/step_breakdown.py > $OUT/stepbd_${v}_$rep.txt 2>&1
  timeout 200 python tools/step_breakdown.py --reqs 4 --len 100 >> $OUT/stepbd_${v}_$rep.txt 2>&1
  if [ $rep = 1 ]; then
    timeout 120 python tools/k1_trace.py --sizes 4x100,16x1000 --fused > $OUT/trace_$v.txt 2>&1
    timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_fused_step_gpu.py tests/test_dcp_step_gpu.py tests/test_step_graph_gpu.py tests/test_layer_graph_gpu.py tests/test_multiproc_ipc_gpu.py -m gpu -q -x > $OUT/pytest_$v.log 2>&1; echo "rc=$?" >> $OUT/pytest_$v.log
  fi
done; done
cp /tmp/lib_base.so $L
