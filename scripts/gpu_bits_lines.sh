#!/bin/bash
# bench lines of the bitstring configs (with the CPU baseline)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for c in c3 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.log 2>&1
done
python scripts/summarize.py | grep -E "^c3|^c5"
