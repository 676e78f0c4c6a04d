#!/bin/bash
# c2 e2e (host output) vs staging chunk size
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for c in 33554432 16777216 8388608 33554432 16777216 8388608; do
  HSF_HOST_CHUNK_BYTES=$c timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/e.log 2>&1
  python -c "import json; l=[x for x in open('/tmp/e.log') if x.startswith('{')]; d=json.loads(l[-1]); print('c2 chunk=$c', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3))"
done
