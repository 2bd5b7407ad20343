#!/bin/bash
# gpurun: selected GPU tests.  bash tools/gpu_quick.sh TAG "pytest-args"
set -u
TAG=$1; shift
mkdir -p gpurun_out
timeout 1200 python -m pytest -m gpu -q -x "$@" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
