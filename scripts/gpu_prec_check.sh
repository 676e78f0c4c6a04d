#!/bin/bash
# precision modes: parity subset + c2 bench per precision
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -x -q -k "bf16 or precision or c2 or tail or c4_full" > gpurun_out/quick_tests.log 2>&1; tail -1 gpurun_out/quick_tests.log
grep -E "Error|assert" gpurun_out/quick_tests.log | head -5
for pr in bf16x3 bf16x6 tf32x3; do
  timeout 600 python bench.py --config c2 --precision $pr --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_$pr.log 2>&1
done
python scripts/summarize.py
