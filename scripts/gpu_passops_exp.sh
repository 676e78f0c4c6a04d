#!/bin/bash
# ops-per-pass cap (smaller generated kernels on long op chains)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for cfg in ${CFGS:-c3 c5 q32-1 c2}; do
  for m in ${CAPS:-0 24 48}; do
    HSF_MAX_PASS_OPS=$m timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > /tmp/po.log 2>&1
    python -c "import json; l=[x for x in open('/tmp/po.log') if x.startswith('{')]; d=json.loads(l[-1]); print('$cfg cap=$m', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()}, d['gpu_launches'])"
  done
done
