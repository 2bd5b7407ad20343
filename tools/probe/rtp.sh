cp tools/probe/_bin/plprof/libdcp_b200.so paper_2605_21100_b200/_build/libdcp_b200.so
timeout 300 python tools/planner_prof.py > gpurun_out/rtprof.txt 2>&1
