#!/bin/bash
# q33-3 (swapped path-sum + row light cone): launch list with DRAM bytes, ncu --set full of the GEMM
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r01s}
python -m paper_2502_06959_b200.build > /dev/null
timeout 300 python scripts/prof_once.py q33-3 auto 2 > gpurun_out/plain_q33.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_q33-3.csv python scripts/prof_once.py q33-3 auto 2 > gpurun_out/ncu_launch_q33.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -s 1 -c 1 \
  -o gpurun_out/${TAG}_q33_gemm python scripts/prof_once.py q33-3 auto 2 > gpurun_out/ncu_full_q33.log 2>&1
echo "ncu gemm rc=$?"
for f in gpurun_out/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$f" --page details > "${f%.ncu-rep}_details.txt" 2>/dev/null
  rm -f "$f"
done
cat gpurun_out/plain_q33.log | tail -1
