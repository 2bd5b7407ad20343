#!/bin/bash
# gpurun: K10 MLA — parity tests, bench, ncu launch list + one full capture.  bash tools/gpu_mla.sh TAG [full]
set -u
TAG=${1:-mla}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python -m pytest tests/test_mla_gpu.py -q -x > $OUT/pytest_mla_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_mla_$TAG.log
timeout 300 python bench_mla.py --steps 100 > $OUT/bench_mla_$TAG.jsonl 2> $OUT/bench_mla_$TAG.err
if [ "${2:-}" = "full" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_mla_$TAG.csv \
      python bench_mla.py --steps 5 --warmup 3 --only cfg2 > $OUT/ncu_launch_mla_$TAG.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_decode_kernel -s 3 -c 1 \
      -o $OUT/k10_$TAG -f python bench_mla.py --steps 2 --warmup 3 --only cfg2 > $OUT/ncu_full_mla_$TAG.log 2>&1
fi
echo done
