#!/bin/bash
# fused reduce-scatter: GPU tests + a 1-GPU bench in fused_rs mode (one shard)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
grep -E "^E |FAILED" gpurun_out/gpu_tests.log | head -5
timeout 600 python bench.py --collective fused_rs --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_fused.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.log 2>&1
python scripts/summarize.py
