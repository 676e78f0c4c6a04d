#!/bin/bash
# c3 e2e (host buffers) vs pass cap
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for m in 128 40 128 40; do
  HSF_MAX_PASS_OPS=$m timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/e.log 2>&1
  python -c "import json; l=[x for x in open('/tmp/e.log') if x.startswith('{')]; d=json.loads(l[-1]); print('c3 cap=$m', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), d['gpu_launches'])"
done
