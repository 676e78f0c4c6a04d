#!/bin/bash
# c4 GEMM experiments: epilogue chunk rotation on/off
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "bf16 or c4_full or accumulate" > gpurun_out/quick_tests.log 2>&1; tail -1 gpurun_out/quick_tests.log
for r in 1 0; do
  HSF_TC_ROT=$r timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_rot$r.log 2>&1
done
HSF_TC_ROT=1 timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
python scripts/summarize.py
