#!/bin/bash
# c4: grouped raster size
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for g in 16 4 64 16; do
  HSF_TC_GROUP_M=$g timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > /tmp/c4.log 2>&1
  python -c "import json; l=[x for x in open('/tmp/c4.log') if x.startswith('{')]; d=json.loads(l[-1]); print('c4 group=$g', round(d['ms_per_step'],3), round(d['phase_ms']['core'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
