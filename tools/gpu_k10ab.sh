#!/bin/bash
# K10 A/B: bench_mla + pair-0 trace for the product build and each tools/probe/_bin/k10_* variant;
# parity (tests/test_mla_gpu.py) for each variant.   bash tools/gpu_k10ab.sh TAG [variants...]
set -u
TAG=$1; shift
OUT=gpurun_out/k10ab_$TAG
mkdir -p $OUT
L=paper_2605_21100_b200/_build/libdcp_b200.so
cp $L /tmp/lib_base.so
for v in base "$@"; do
  if [ $v != base ]; then cp tools/probe/_bin/k10_$v/libdcp_b200.so $L || { echo "missing variant k10_$v" > $OUT/bench_$v.jsonl; continue; }; else cp /tmp/lib_base.so $L; fi
  timeout 300 python bench_mla.py --steps 50 > $OUT/bench_$v.jsonl 2>&1
  timeout 120 python tools/mla_trace.py > $OUT/trace_$v.txt 2>&1
  if [ $v != base ] && [ -z "${NOTEST:-}" ]; then timeout 300 python -m pytest tests/test_mla_gpu.py -m gpu -q -x > $OUT/pytest_$v.log 2>&1; echo "rc=$?" >> $OUT/pytest_$v.log; fi
done
cp /tmp/lib_base.so $L
for v in base "$@"; do echo "== $v"; python -c "
import json
for l in open('$OUT/bench_$v.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['workload'], round(d['ms_per_step'],4), round(d['roofline_frac'],3))
"; tail -5 $OUT/trace_$v.txt; tail -1 $OUT/pytest_$v.log 2>/dev/null; done
