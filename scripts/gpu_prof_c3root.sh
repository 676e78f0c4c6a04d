#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python scripts/prof_once.py c3 auto 1 > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hsf_jit" -s 2 -c 1 \
  -o gpurun_out/r01h_c3_root python scripts/prof_once.py c3 auto 1 > gpurun_out/ncu_full_c3.log 2>&1
echo "ncu rc=$?"
for f in gpurun_out/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$f" --page details > "${f%.ncu-rep}_details.txt" 2>/dev/null
  ncu -i "$f" --page source --csv > "${f%.ncu-rep}_source.csv" 2>/dev/null
  rm -f "$f"
done
