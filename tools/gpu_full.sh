#!/bin/bash
# gpurun: full round check — GPU tests, smoke, bench, DCP bench, ncu launch list + full capture of K1.
set -u
TAG=${1:-full}
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" >> $OUT/bench_$TAG.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 900 python bench_dcp.py --steps 300 > $OUT/bench_dcp_$TAG.json 2> $OUT/bench_dcp_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-mla > $OUT/ncu_launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:splitkv_decode -s 3 -c 1 \
    -o $OUT/k1_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-mla > $OUT/ncu_full_$TAG.log 2>&1
echo done
