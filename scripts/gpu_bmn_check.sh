#!/bin/bash
# MN-major B operand: parity subset + c2/c4 bench, MN-major vs K-major
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -x -q -k "tail or bf16 or c2 or c4_full or accumulate or partition" > gpurun_out/quick_tests.log 2>&1; tail -3 gpurun_out/quick_tests.log
for v in 1 0; do
  HSF_TC_BMN=$v timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_bmn$v.log 2>&1
done
HSF_TC_BMN=1 timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_bmn1.log 2>&1
python scripts/summarize.py
