#!/bin/bash
# A/B: c2 bench of an older build (old_wt/) vs the current tree, interleaved
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for i in 1 2; do
  for t in old_wt .; do
    (cd $t && timeout 600 python bench.py --config ${CFG:-c2} --steps 20 --warmup 5 --no-cpu-baseline > /tmp/ab.log 2>&1)
    python -c "import json; l=[x for x in open('/tmp/ab.log') if x.startswith('{')]; d=json.loads(l[-1]); print('$t', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})"
  done
done
