#!/bin/bash
# gpurun: K10 timings for a list of DCP_MLA_DBG values.  bash tools/gpu_mla_dbg.sh TAG PAGE "D1 D2 ..."
set -u
TAG=$1; P=$2; DS=$3
mkdir -p gpurun_out
for D in $DS; do
  DCP_MLA_PAGE=$P DCP_MLA_DBG=$D timeout 60 python bench_mla.py --steps 50 > gpurun_out/ab_${TAG}_p${P}_d$D.jsonl 2>&1
done
echo done
