#!/bin/bash
# full GPU suite, then the q configs' bench lines (phase breakdown)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2502_06959_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -rfs > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
for cfg in q30-1 q32-1 q33-3; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bq_${cfg}.log 2>&1
  python -c "import json; l=[x for x in open('gpurun_out/bq_${cfg}.log') if x.startswith('{')]; d=json.loads(l[-1]); print('$cfg', d['ms_per_step'], d['phase_ms'], d['roofline'].get('kernel'), d['roofline']['frac'])"
done
