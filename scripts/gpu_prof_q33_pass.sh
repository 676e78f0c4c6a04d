#!/bin/bash
# q33-3: ncu --set full of half B's leaf pass (operand store) -- the 6th hsf_jit_pass launch
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r01s}
python -m paper_2502_06959_b200.build > /dev/null
timeout 300 python scripts/prof_once.py q33-3 auto 1 > gpurun_out/plain_q33.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hsf_jit_pass" -s 5 -c 1 \
  -o gpurun_out/${TAG}_q33_bleaf python scripts/prof_once.py q33-3 auto 1 > gpurun_out/ncu_full_q33b.log 2>&1
echo "ncu rc=$?"
for f in gpurun_out/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$f" --page details > "${f%.ncu-rep}_details.txt" 2>/dev/null
  ncu -i "$f" --page source --csv > "${f%.ncu-rep}_source.csv" 2>/dev/null
  rm -f "$f"
done
