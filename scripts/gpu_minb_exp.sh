#!/bin/bash
# heavy simulator passes: __launch_bounds__ min blocks 2 vs 3
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for cfg in ${CFGS:-q33-3 q32-1 c5 c3 c2}; do
  for mb in ${MBS:-2 3}; do
    HSF_JIT_HEAVY_MINB=$mb timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/mb_${cfg}_$mb.log 2>&1
    python -c "import json; l=[x for x in open('gpurun_out/mb_${cfg}_$mb.log') if x.startswith('{')]; d=json.loads(l[-1]); print('$cfg minb=$mb', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
  done
done
