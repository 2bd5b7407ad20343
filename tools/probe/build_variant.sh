#!/bin/bash
# Build a variant of libdcp_b200.so with extra nvcc -D flags on one TU into
# tools/probe/_bin/<name>/ (A/B experiments; run after the product build).
#   tools/probe/build_variant.sh NAME TU.cu -DFOO=0 ...
set -eu
cd "$(dirname "$0")/../.."
NAME=$1; TU=$2; shift 2
B=paper_2605_21100_b200/_build
O=tools/probe/_bin/$NAME
mkdir -p $O
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -ccbin /usr/bin/g++ \
    -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -Ipaper_2605_21100_b200/csrc \
    "$@" -c paper_2605_21100_b200/csrc/$TU -o $O/$TU.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -cudart static \
    -o $O/libdcp_b200.so $(ls $B/*.o | grep -v "/$TU.o") $O/$TU.o -lrt
echo built $O/libdcp_b200.so
