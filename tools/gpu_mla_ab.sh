#!/bin/bash
# gpurun: K10 bottleneck matrix (page x DCP_MLA_DBG) + parity.  bash tools/gpu_mla_ab.sh TAG
set -u
TAG=$1
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_mla_gpu.py -q -x > gpurun_out/pytest_mla_$TAG.log 2>&1
for P in 16 64; do for D in 0 1 2 3; do
  DCP_MLA_PAGE=$P DCP_MLA_DBG=$D timeout 60 python bench_mla.py --steps 50 > gpurun_out/ab_${TAG}_p${P}_d$D.jsonl 2>&1
done; done
echo done
