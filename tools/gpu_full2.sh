#!/bin/bash
# gpurun: full round-2 check — all GPU tests, smoke, bench (N=1), reference arm, DCP bench, MoE bench,
# graph bench, trace bench (whole-layer TPOT), 2-rank bench emulation, ncu launch list + K1 full capture.
set -u
TAG=${1:-full2}
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=10 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" >> $OUT/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 900 python bench_dcp.py --steps 1000 > $OUT/bench_dcp_$TAG.jsonl 2> $OUT/bench_dcp_$TAG.err
timeout 300 python bench_moe.py --steps 20 > $OUT/bench_moe_$TAG.jsonl 2>&1
timeout 300 python bench_graph.py > $OUT/bench_graph_$TAG.json 2>&1
timeout 900 python bench_trace.py --duration 10 --rate 16 > $OUT/bench_trace_$TAG.jsonl 2> $OUT/bench_trace_$TAG.err
DCP_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > $OUT/bench_multi2_$TAG.json 2> $OUT/bench_multi2_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-mla --no-moe --no-dcp > $OUT/ncu_launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:splitkv_decode -s 3 -c 1 \
    -o $OUT/k1_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-mla --no-moe --no-dcp > $OUT/ncu_full_$TAG.log 2>&1
echo done
