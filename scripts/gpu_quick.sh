cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -rf > gpurun_out/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 300 python scripts/prof_once.py c2 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
  python scripts/prof_once.py c2 > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/gpu_tests.log
python - <<'PY'
import json, csv
for l in open('gpurun_out/bench.log'):
    if l.startswith('{'): d=json.loads(l); print('ms/step', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})
with open('gpurun_out/launches.csv') as f:
    lines=[l for l in f if l.startswith('"')]
rows=[x for x in csv.DictReader(lines) if x['Metric Name']=='gpu__time_duration.sum']
for x in rows[:30]:
    print(x['ID'], x['Kernel Name'][:30], x['Stream'], x['Block Size'], x['Grid Size'], float(x['Metric Value'])/1e3)
PY
