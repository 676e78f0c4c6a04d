cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python scripts/prof_once.py c4 auto 1 16 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"tc_gemm" -c 1 \
  -o gpurun_out/r01c_c4_gemm python scripts/prof_once.py c4 auto 1 16 > gpurun_out/ncu_full_c4.log 2>&1
echo "ncu c4 rc=$?"
timeout 300 python scripts/prof_once.py c5 auto 1 > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r01c_launches_c5.csv python scripts/prof_once.py c5 auto 1 > gpurun_out/ncu_launch_c5.log 2>&1
echo "launch c5 rc=$?"
for f in gpurun_out/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$f" --page details > "${f%.ncu-rep}_details.txt" 2>/dev/null
  rm -f "$f"
done
cat gpurun_out/plain_c4.log gpurun_out/plain_c5.log
