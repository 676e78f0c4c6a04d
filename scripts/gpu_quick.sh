#!/bin/bash
# Quick loop: a pytest -k selection + benches of the given configs.
#   gpurun -- 'bash scripts/gpu_quick.sh "<pytest -k expr>" c2 c4'
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
K="$1"; shift
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -rf -k "$K" > gpurun_out/quick_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/quick_tests.log
tail -3 gpurun_out/quick_tests.log
for c in "$@"; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  echo "bench $c rc=$?" >> gpurun_out/bench_$c.log
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
for l in open(f"gpurun_out/bench_{c}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        r = d["roofline"]
        print(c, "ms/step %.3f" % d["ms_per_step"], {k: round(v, 3) for k, v in d["phase_ms"].items()},
              r["bound"], "%.1f %s frac %.3f" % (r["achieved"], r["unit"], r["frac"]))
PY
  tail -1 gpurun_out/bench_$c.log
done
