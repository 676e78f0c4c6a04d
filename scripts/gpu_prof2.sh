cd $GRAFT_REPO_ROOT
timeout 300 python scripts/prof_once.py c2 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hsf_pass" --launch-skip 24 --launch-count 1 \
  -o gpurun_out/prof_alev2 python scripts/prof_once.py c2 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
