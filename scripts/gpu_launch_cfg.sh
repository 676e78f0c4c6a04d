#!/bin/bash
# launch list of one hsf_run of a config:  bash scripts/gpu_launch_cfg.sh c3 tag
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
C=${1:-c3}; TAG=${2:-r01g}
timeout 300 python scripts/prof_once.py $C auto 1 > gpurun_out/plain_$C.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_$C.csv python scripts/prof_once.py $C auto 1 > gpurun_out/ncu_launch_$C.log 2>&1
echo rc=$?
