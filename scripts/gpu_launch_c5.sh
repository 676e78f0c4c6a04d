cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python scripts/prof_once.py c5 auto 1 > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r01e_launches_c5.csv python scripts/prof_once.py c5 auto 1 > gpurun_out/ncu_launch_c5.log 2>&1
echo rc=$?
