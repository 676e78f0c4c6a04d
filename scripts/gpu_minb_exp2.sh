#!/bin/bash
# simulator pass __launch_bounds__ min blocks: heavy/light combinations
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for cfg in q33-3 q32-1 c5 c3 q30-1; do
  for hl in "4 3" "4 4" "5 4" "4 5"; do
    set -- $hl
    HSF_JIT_HEAVY_MINB=$1 HSF_JIT_LIGHT_MINB=$2 timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > /tmp/mb.log 2>&1
    python -c "import json; l=[x for x in open('/tmp/mb.log') if x.startswith('{')]; d=json.loads(l[-1]); print('$cfg h=$1 l=$2', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
  done
done
