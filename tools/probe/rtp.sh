# K7 / K6: planner tests + timing (normal build), then the DCP_PLANNER_PROF build's phase stamps
# (build the profiling library first: bash tools/probe/build_prof.sh)
timeout 900 python -m pytest -m gpu -q -x tests/test_planner_gpu.py tests/test_dcp_step_gpu.py tests/test_decode_growth_gpu.py tests/test_dropin_gpu.py > gpurun_out/pytest_rtp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rtp.log
for r in 1 2; do timeout 300 python tools/planner_prof.py >> gpurun_out/rtprof_t.txt 2>&1; done
cp tools/probe/_bin/plprof/libdcp_b200.so paper_2605_21100_b200/_build/libdcp_b200.so
timeout 300 python tools/planner_prof.py > gpurun_out/rtprof.txt 2>&1
