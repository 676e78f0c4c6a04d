#!/bin/bash
# Launch lists + small ncu --set full captures; keeps gpurun_out/ < 64 MiB.
#   gpurun -- 'bash scripts/gpu_prof.sh <tag>'
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r01}
for c in c5 c2; do
timeout 300 python scripts/prof_once.py $c auto 1 > gpurun_out/plain_once_$c.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_$c.csv python scripts/prof_once.py $c auto 1 > gpurun_out/ncu_launch_$c.log 2>&1
echo "launch list $c rc=$?"
done
timeout 300 python scripts/prof_once.py c5 auto 1 > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hsf_pass" -s 6 -c 1 \
  -o gpurun_out/${TAG}_c5_bleaf python scripts/prof_once.py c5 auto 1 > gpurun_out/ncu_full_c5.log 2>&1
echo "ncu c5 rc=$?"
timeout 300 python scripts/prof_once.py c4 auto 1 16 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -c 1 \
  -o gpurun_out/${TAG}_c4_gemm python scripts/prof_once.py c4 auto 1 16 > gpurun_out/ncu_full_c4.log 2>&1
echo "ncu c4 rc=$?"
for f in gpurun_out/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$f" --page details > "${f%.ncu-rep}_details.txt" 2>/dev/null
  ncu -i "$f" --page source --csv > "${f%.ncu-rep}_source.csv" 2>/dev/null
  if [ $(stat -c %s "$f") -gt 15000000 ]; then rm -f "$f"; fi
done
cat gpurun_out/plain_*.log
du -sh gpurun_out
