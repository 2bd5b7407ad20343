#!/bin/bash
# gpurun: one ncu --set full capture of the K10 kernel (cfg2-shaped MLA).  bash tools/gpu_mla_ncu.sh TAG [only]
set -u
TAG=$1
ONLY=${2:-cfg2}
mkdir -p gpurun_out
DCP_MLA_DBG=${DBG:-0} timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_decode_kernel -s 3 -c 1 \
    -o gpurun_out/k10_$TAG -f python bench_mla.py --steps 2 --warmup 3 --only $ONLY > gpurun_out/ncu_full_mla_$TAG.log 2>&1
echo done
