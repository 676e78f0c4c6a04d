#!/bin/bash
# simulator-side changes: the parity tests touching the trees + benches c3 c5 c2
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -rf -k "twins or random or tile or hoist or interpreter or c3 or c5 or table2 or partition or fold or graph" > gpurun_out/quick_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/quick_tests.log
for c in c3 c5 c2 q33-3; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
python scripts/summarize.py
