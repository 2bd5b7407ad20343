#!/bin/bash
# gpurun: K1 small-batch fixed cost (events + graphs) and an ncu full capture of a 4x100 launch.
set -u
TAG=${1:-r2d}
mkdir -p gpurun_out
timeout 300 python tools/probe_k1_small.py > gpurun_out/k1small_$TAG.jsonl 2> gpurun_out/k1small_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:splitkv_decode -s 15 -c 1 \
    -o gpurun_out/k1small_$TAG -f python tools/probe_k1_small.py --sizes 4x100 --iters 20 > gpurun_out/k1small_ncu_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:splitkv_decode -s 15 -c 1 \
    -o gpurun_out/k1med_$TAG -f python tools/probe_k1_small.py --sizes 16x1000 --iters 20 >> gpurun_out/k1small_ncu_$TAG.log 2>&1
echo done
