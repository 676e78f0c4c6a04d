#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -rf -k "bits or c5 or c3 or fold or table2 or hoist or interpreter or accumulate or graph or single" > gpurun_out/quick_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/quick_tests.log
for c in c5 c3; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
python scripts/summarize.py
