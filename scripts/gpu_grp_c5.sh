#!/bin/bash
# c5: grouped (bucketed) gather forced vs per-sample gather
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for g in 0 1 0 1; do
  HSF_GROUPED_GATHER=$g timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/g.log 2>&1
  python -c "import json; l=[x for x in open('/tmp/g.log') if x.startswith('{')]; d=json.loads(l[-1]); print('c5 grouped=$g', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
done
