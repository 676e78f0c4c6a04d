#!/bin/bash
# narrow-N swapped GEMM with more stages: parity + q benches
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "swapped or table2 or accumulate or chunked" > gpurun_out/ns_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/ns_tests.log
for cfg in q32-1 q33-3 q30-1; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > /tmp/n.log 2>&1
  python -c "import json; l=[x for x in open('/tmp/n.log') if x.startswith('{')]; d=json.loads(l[-1]); print('$cfg', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
done
