#!/bin/bash
# bitstring path: parity subset + c3/c5 bench, grouped gather on/off
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "bits or c3 or c5 or fold or partition or graph or grouped or transposed or edge" > gpurun_out/quick_tests.log 2>&1; tail -1 gpurun_out/quick_tests.log
grep -E "^E |FAILED" gpurun_out/quick_tests.log | head -5
for c in c3 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_grp.log 2>&1
  HSF_GROUPED_GATHER=0 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_plain.log 2>&1
done
python scripts/summarize.py
