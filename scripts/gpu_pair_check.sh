#!/bin/bash
# Guarded first run of the CTA-pair GEMM: tensor-core tests under a short timeout.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 240 python -m pytest tests -m gpu -x -q --timeout 200 -rf -k "bf16 or accumulate or c2_full or c4_full or host_output" > gpurun_out/pair_tests.log 2>&1
echo "pair tests rc=$?" >> gpurun_out/pair_tests.log
tail -4 gpurun_out/pair_tests.log
if grep -q "pair tests rc=0" gpurun_out/pair_tests.log; then
  timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
  HSF_TC_PAIR=0 timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_single.log 2>&1
  timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
  python scripts/summarize.py
  python - <<'PY'
import json
for f in ["gpurun_out/bench_c2_single.log"]:
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); print("single-CTA c2", round(d["ms_per_step"], 3), round(d["phase_ms"]["core"], 3))
PY
fi
