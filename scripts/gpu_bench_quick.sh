cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in c2 c5 q30-1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; done
python scripts/summarize.py
python - <<'PY'
import json
for c in ["c2","c5","q30-1"]:
    for l in open(f"gpurun_out/bench_{c}.log"):
        if l.startswith("{"): d=json.loads(l); print(c, json.dumps(d["e2e"])[:300], d["gpu_launches"])
PY
