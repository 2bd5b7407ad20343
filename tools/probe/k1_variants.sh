# bench.py (K1 only) for the base lib and each variant, interleaved twice
set -u
cp paper_2605_21100_b200/_build/libdcp_b200.so /tmp/base.so
for rep in 1 2; do
for v in base "$@"; do
  if [ "$v" != base ]; then cp tools/probe/_bin/$v/libdcp_b200.so paper_2605_21100_b200/_build/libdcp_b200.so; fi
  timeout 200 python bench.py --no-cpu-baseline --no-mla --steps 300 > gpurun_out/k1v_${v}_$rep.json 2>/dev/null
  cp /tmp/base.so paper_2605_21100_b200/_build/libdcp_b200.so
done; done
