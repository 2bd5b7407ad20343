# planner: parity tests, timing of the normal build, then the DCP_PLANNER_PROF build (printf section cycles)
# (build the profiling library first: bash tools/probe/build_prof.sh)
timeout 900 python -m pytest -m gpu -q -x tests/test_planner_gpu.py tests/test_dropin_gpu.py tests/test_decode_growth_gpu.py tests/test_dcp_step_gpu.py tests/test_step_graph_gpu.py > gpurun_out/pytest_$1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$1.log
for r in 1 2; do timeout 300 python tools/planner_prof.py >> gpurun_out/planner_prof_$1.txt 2>&1; done
cp tools/probe/_bin/plprof/libdcp_b200.so paper_2605_21100_b200/_build/libdcp_b200.so
timeout 300 python tools/planner_prof.py >> gpurun_out/planner_prof_$1.txt 2>&1
