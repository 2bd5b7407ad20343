#!/bin/bash
# Build the DCP_PLANNER_PROF variant of libdcp_b200.so (planner / routing phase stamps via
# printf) into tools/probe/_bin/plprof/, for tools/probe/plp.sh and rtp.sh.  Run after
# `python -m paper_2605_21100_b200.build` (it links the other objects from _build/).
set -eu
cd "$(dirname "$0")/../.."
B=paper_2605_21100_b200/_build
mkdir -p tools/probe/_bin/plprof
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -ccbin /usr/bin/g++ \
    -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -Ipaper_2605_21100_b200/csrc \
    -DDCP_PLANNER_PROF -c paper_2605_21100_b200/csrc/capi_planner.cu -o tools/probe/_bin/plprof/capi_planner.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -cudart static \
    -o tools/probe/_bin/plprof/libdcp_b200.so $(ls $B/*.o | grep -v capi_planner) tools/probe/_bin/plprof/capi_planner.o -lrt
echo built tools/probe/_bin/plprof/libdcp_b200.so
