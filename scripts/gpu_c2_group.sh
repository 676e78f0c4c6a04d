#!/bin/bash
# c2: tile raster (M-fastest vs grouped)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for g in 0 4 8 0 4 8; do
  HSF_TC_GROUP_M=$g timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > /tmp/g.log 2>&1
  python -c "import json; l=[x for x in open('/tmp/g.log') if x.startswith('{')]; d=json.loads(l[-1]); print('c2 group=$g', round(d['ms_per_step'],4), round(d['phase_ms']['core'],4))"
done
