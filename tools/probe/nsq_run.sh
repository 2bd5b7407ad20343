set -u
cp paper_2605_21100_b200/_build/libdcp_b200.so /tmp/base.so
for n in 8 12; do
  cp tools/probe/_bin/nsq$n/libdcp_b200.so paper_2605_21100_b200/_build/libdcp_b200.so
  bash tools/gpu_mla_dbg.sh n$n 16 "0 3"; bash tools/gpu_mla_dbg.sh n$n 64 "0 3"
done
cp /tmp/base.so paper_2605_21100_b200/_build/libdcp_b200.so
