#!/bin/bash
# c4 GEMM experiment: pipeline depth <3,1> vs <2,2>
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
HSF_TC_CFG=16 timeout 300 python -m pytest tests -m gpu -x -q -k "bf16 or c4_full" > gpurun_out/quick_tests.log 2>&1; tail -1 gpurun_out/quick_tests.log
for cfg in 16 22; do
  HSF_TC_CFG=$cfg timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_cfg$cfg.log 2>&1
done
python scripts/summarize.py
