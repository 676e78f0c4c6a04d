#!/bin/bash
# c4 GEMM experiment: LSU vs TMA-store epilogue
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
HSF_TC_LSU=1 timeout 300 python -m pytest tests -m gpu -x -q -k "bf16 or c4_full or c2_full" > gpurun_out/quick_tests.log 2>&1; tail -1 gpurun_out/quick_tests.log
for v in 1 0; do
  HSF_TC_LSU=$v timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_lsu$v.log 2>&1
  HSF_TC_LSU=$v timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_lsu$v.log 2>&1
done
python scripts/summarize.py
