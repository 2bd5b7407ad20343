# K7 timing: planner_prof with the current build (3 runs), then the A/B build in $2 if given
timeout 900 python -m pytest -m gpu -q -x tests/test_planner_gpu.py tests/test_dcp_step_gpu.py tests/test_decode_growth_gpu.py tests/test_dropin_gpu.py tests/test_step_graph_gpu.py > gpurun_out/pytest_$1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$1.log
for r in 1 2 3; do timeout 300 python tools/planner_prof.py >> gpurun_out/rt_$1.txt 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:routing --log-file gpurun_out/rt_$1_launch.csv python tools/planner_prof.py > /dev/null 2>&1
