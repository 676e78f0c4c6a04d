#!/bin/bash
# One GPU round trip: parity tests, smoke, bench (c2 default), launch list.
# Usage (from this container):  gpurun --timeout 1500 -- 'bash scripts/gpu_check.sh'
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -rf > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; tail -2 gpurun_out/bench.log
