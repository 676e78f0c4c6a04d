#!/bin/bash
# c2 with different tail-fold prefix budgets
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for b in 16777216 4194304 1048576 262144; do
  HSF_TAIL_PREFIX_BYTES=$b timeout 300 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_tb$b.log 2>&1
done
python scripts/summarize.py
