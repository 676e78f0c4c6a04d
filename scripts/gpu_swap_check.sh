#!/bin/bash
# swapped prefix path-sum: parity, then q-config benches with the swap off / on
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "swapped or table2 or accumulate or chunked" > gpurun_out/swap_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/swap_tests.log
for cfg in q30-1 q32-1 q33-3; do
  for s in 0 1; do
    HSF_TC_SWAP=$s timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/swap_${cfg}_$s.log 2>&1
    echo "$cfg swap=$s: $(python -c "import json,sys; l=[x for x in open('gpurun_out/swap_${cfg}_$s.log') if x.startswith('{')]; d=json.loads(l[-1]); print(d['ms_per_step'], d.get('e2e',{}).get('value'))" 2>&1 | tail -1)"
  done
done
