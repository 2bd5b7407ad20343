#!/bin/bash
# gpurun: routed small-step breakdown (events + ncu kernel durations), MoE bench, 2-rank bench emulation.
set -u
TAG=${1:-r2c}
mkdir -p gpurun_out
for a in "--reqs 16 --len 1000" "--reqs 64 --len 2048" "--reqs 4 --len 100"; do
  timeout 300 python tools/step_breakdown.py $a >> gpurun_out/breakdown_$TAG.jsonl 2>> gpurun_out/breakdown_$TAG.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/breakdown_launches_$TAG.csv \
   python tools/step_breakdown.py --iters 20 > /dev/null 2>&1
timeout 300 python bench_moe.py --steps 20 > gpurun_out/bench_moe_$TAG.jsonl 2>&1
DCP_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_multi2_$TAG.json 2> gpurun_out/bench_multi2_$TAG.err
echo done
