#!/bin/bash
# 3M (Gauss) GEMM: parity + c2 bench with / without
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 300 python -m pytest tests -m gpu -x -q -s -k "gauss" > gpurun_out/quick_tests.log 2>&1; tail -1 gpurun_out/quick_tests.log
grep -E "^E |FAILED|3M max" gpurun_out/quick_tests.log | head -6
for v in 1 0; do
  HSF_TC_3M=$v timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_3m$v.log 2>&1
done
python scripts/summarize.py
