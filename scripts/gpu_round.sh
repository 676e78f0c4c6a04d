cd $GRAFT_REPO_ROOT
timeout 300 python scripts/prof_once.py c2 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hsf_pass" --launch-skip 11 --launch-count 2 \
  -o gpurun_out/prof_qft2 python scripts/prof_once.py c2 > gpurun_out/ncu_full.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hsf_pass" --launch-skip 23 --launch-count 1 \
  -o gpurun_out/prof_alev python scripts/prof_once.py c2 > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/ncu_full.log
