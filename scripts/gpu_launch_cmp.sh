#!/bin/bash
# launch lists of one config with and without an env toggle:  bash scripts/gpu_launch_cmp.sh c3 HSF_NO_CLUSTER
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
C=${1:-c3}; V=${2:-HSF_NO_CLUSTER}
timeout 300 python scripts/prof_once.py $C auto 1 > gpurun_out/plain_$C.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/cmp_on_$C.csv python scripts/prof_once.py $C auto 1 > gpurun_out/ncu_on.log 2>&1
env $V=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/cmp_off_$C.csv python scripts/prof_once.py $C auto 1 > gpurun_out/ncu_off.log 2>&1
echo rc=$?
