#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 500 -rf -k "bucket or c5 or bits or accumulate" > gpurun_out/quick_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
HSF_NO_SORT=1 timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_nosort.log 2>&1
python scripts/summarize.py
