#!/bin/bash
# c5 launch list with DRAM bytes (one run)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r01u}
python -m paper_2502_06959_b200.build > /dev/null
timeout 300 python scripts/prof_once.py ${CFG:-c5} auto 1 > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_${CFG:-c5}.csv python scripts/prof_once.py ${CFG:-c5} auto 1 > gpurun_out/ncu_launch_c5.log 2>&1
echo "launch list rc=$?"
