#!/bin/bash
# round end: full GPU suite, smoke, bench line of every config
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -rf > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.log 2>&1
for c in c1 c3 c5 q30-1 q32-1 q33-3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.log 2>&1
done
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1
python scripts/summarize.py | grep -v "_sk\|_tc"
