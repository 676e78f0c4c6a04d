#!/bin/bash
# c4 GEMM experiment: grouped raster
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
HSF_TC_GROUP_M=8 timeout 300 python -m pytest tests -m gpu -x -q -k "bf16 or c4_full" > gpurun_out/quick_tests.log 2>&1; tail -1 gpurun_out/quick_tests.log
for g in 0 4 8 16 32; do
  HSF_TC_GROUP_M=$g timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_g$g.log 2>&1
done
HSF_TC_GROUP_M=8 timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_g8.log 2>&1
python scripts/summarize.py
