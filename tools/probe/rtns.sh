cp tools/probe/_bin/rtns/libdcp_b200.so paper_2605_21100_b200/_build/libdcp_b200.so
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:routing_rows --log-file gpurun_out/rtns_launch.csv python tools/planner_prof.py > gpurun_out/rtns.txt 2>&1
