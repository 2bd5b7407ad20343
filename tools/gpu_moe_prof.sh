#!/bin/bash
# gpurun: MoE kernels launch list + one full ncu capture of K4.  bash tools/gpu_moe_prof.sh TAG
set -u
TAG=${1:-moe}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/moe_launches_$TAG.csv \
    python bench_moe.py --steps 3 --warmup 1 > gpurun_out/moe_ncu_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moe_dispatch -s 40 -c 1 \
    -o gpurun_out/moe_disp_$TAG -f python bench_moe.py --steps 3 --warmup 1 >> gpurun_out/moe_ncu_$TAG.log 2>&1
echo done
