#!/bin/bash
# simulator change: full GPU suite + sim-heavy benches
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
grep -E "^E |FAILED" gpurun_out/gpu_tests.log | head -5
for c in c5 c3 q33-3 q32-1 c2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
python scripts/summarize.py
