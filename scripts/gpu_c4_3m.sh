#!/bin/bash
# c4: 4-real-GEMM x3 vs 3M, with clocks
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
for m in 1 0 1; do
  HSF_TC_LSU=0 HSF_TC_3M=$m timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > /tmp/c4.log 2>&1
  python -c "import json; l=[x for x in open('/tmp/c4.log') if x.startswith('{')]; d=json.loads(l[-1]); print('c4 3m=$m', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()}, d['clocks'])"
done
nvidia-smi -q -d POWER | grep -iE "limit|draw" | head -6
