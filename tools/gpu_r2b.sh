#!/bin/bash
# gpurun: new protocol/IPC tests, MoE bench, multi-rank bench emulated on one GPU.  bash tools/gpu_r2b.sh TAG
set -u
TAG=${1:-r2b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multiproc_ipc_gpu.py tests/test_exchange_protocol_gpu.py tests/test_moe_gpu.py tests/test_cfg1_gpu.py -m gpu -q -rA -s > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench_moe.py --steps 20 > gpurun_out/bench_moe_$TAG.jsonl 2>&1; echo "moe rc=$?" >> gpurun_out/bench_moe_$TAG.jsonl
DCP_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_multi2_$TAG.json 2> gpurun_out/bench_multi2_$TAG.err; echo "multi rc=$?" >> gpurun_out/bench_multi2_$TAG.err
tail -3 gpurun_out/pytest_$TAG.log
