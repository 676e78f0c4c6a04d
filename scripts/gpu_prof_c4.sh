#!/bin/bash
# ncu --set full of the c4 GEMM on a 1/16 row slice (same tile shape), raw metrics exported
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r01o}
python -m paper_2502_06959_b200.build > /dev/null
timeout 300 python scripts/prof_once.py c4 auto 2 16 > gpurun_out/plain_c4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -s 1 -c 1 \
  -o gpurun_out/${TAG}_c4_gemm python scripts/prof_once.py c4 auto 2 16 > gpurun_out/ncu_full_c4.log 2>&1
echo "ncu rc=$?"
for f in gpurun_out/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$f" --page details > "${f%.ncu-rep}_details.txt" 2>/dev/null
  rm -f "$f"
done
