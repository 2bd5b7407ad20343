#!/bin/bash
# gpurun: K10 parity tests, bench_mla, and the K10 launch list (decode / scan / merge).
set -u
TAG=${1:-m}
mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q -x tests/test_mla_gpu.py > gpurun_out/pytest_mla_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mla_$TAG.log
timeout 600 python bench_mla.py > gpurun_out/bench_mla_$TAG.jsonl 2> gpurun_out/bench_mla_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:mla_ --log-file gpurun_out/mla_${TAG}_launch.csv python bench_mla.py --steps 4 --warmup 3 > /dev/null 2>&1
echo done
