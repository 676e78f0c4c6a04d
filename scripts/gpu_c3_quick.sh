#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -x -q -k "grouped or bits or c3 or c5" > gpurun_out/quick_tests.log 2>&1; tail -1 gpurun_out/quick_tests.log
for c in c3 c5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_q.log 2>&1; done
python scripts/summarize.py
bash scripts/gpu_launch_cfg.sh c3 ${1:-r01v}
