#!/bin/bash
# gpurun: racecheck over every planner test, then the planner / drop-in / growth / cfg1 parity tests.
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest -q -m gpu -x \
   "tests/test_planner_gpu.py" > gpurun_out/sanitize4_racecheck.log 2>&1; echo "exit=$?" >> gpurun_out/sanitize4_racecheck.log
timeout 900 python -m pytest -m gpu -q -x tests/test_planner_gpu.py tests/test_dropin_gpu.py tests/test_decode_growth_gpu.py tests/test_cfg1_gpu.py > gpurun_out/pytest_s4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_s4.log
