#!/bin/bash
# quick c2: parity subset, bench, launch list
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -x -q -k "tail or bf16 or c2 or accumulate or partition" > gpurun_out/quick_tests.log 2>&1; tail -1 gpurun_out/quick_tests.log
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_q.log 2>&1
python scripts/summarize.py
bash scripts/gpu_launch_cfg.sh c2 ${1:-r01k}
