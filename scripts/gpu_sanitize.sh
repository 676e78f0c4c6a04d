#!/bin/bash
# gpurun -- 'bash scripts/gpu_sanitize.sh memcheck|racecheck|synccheck'
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=${1:-memcheck}
timeout 300 python scripts/sanitize.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_$T.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_$T.log
tail -5 gpurun_out/sanitize_$T.log
