#!/bin/bash
# grouped gather with lane-parallel index loads: parity + c5 / c3
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "bits or grouped or folding or partition or graph or c3 or c5" > gpurun_out/gg_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/gg_tests.log
for cfg in c5 c3 c5 c3; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > /tmp/t.log 2>&1
  python -c "import json; l=[x for x in open('/tmp/t.log') if x.startswith('{')]; d=json.loads(l[-1]); print('$cfg', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
done
