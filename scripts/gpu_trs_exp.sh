#!/bin/bash
# transposed-store leaf pass (bitstring runs) at 4 CTAs/SM heavy passes
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for cfg in c5 c3; do
  for t in 0 1 0 1; do
    HSF_TRANSPOSED_STORE=$t timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > /tmp/t.log 2>&1
    python -c "import json; l=[x for x in open('/tmp/t.log') if x.startswith('{')]; d=json.loads(l[-1]); print('$cfg trs=$t', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
  done
done
