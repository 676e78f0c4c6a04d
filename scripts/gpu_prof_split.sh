#!/bin/bash
# ncu --set full of c2's operand-prep kernels (split_a_mn, split_b_mn)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r01k}
python -m paper_2502_06959_b200.build > /dev/null
timeout 300 python scripts/prof_once.py c2 auto 2 > gpurun_out/plain_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"split_" -s 2 -c 2 \
  -o gpurun_out/${TAG}_c2_split python scripts/prof_once.py c2 auto 2 > gpurun_out/ncu_split.log 2>&1
echo "ncu rc=$?"
for f in gpurun_out/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$f" --page details > "${f%.ncu-rep}_details.txt" 2>/dev/null
  rm -f "$f"
done
