#!/bin/bash
# pytest -m gpu [-k expr] with skip reasons
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -rfs ${1:+-k "$1"} > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -6 gpurun_out/gpu_tests.log
