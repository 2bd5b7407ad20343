# run bench_mla (page 16; DBG values in $DBGS, default "0") + trace for the base lib and each variant dir given
set -u
DBGS=${DBGS:-0}
cp paper_2605_21100_b200/_build/libdcp_b200.so /tmp/base.so
for v in base "$@"; do
  if [ "$v" != base ]; then cp tools/probe/_bin/$v/libdcp_b200.so paper_2605_21100_b200/_build/libdcp_b200.so; fi
  bash tools/gpu_mla_dbg.sh v_$v 16 "$DBGS"
  timeout 60 python tools/mla_trace.py > gpurun_out/trace_v_$v.txt 2>&1
  cp /tmp/base.so paper_2605_21100_b200/_build/libdcp_b200.so
done
