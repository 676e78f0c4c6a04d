#!/bin/bash
# Launch lists + small ncu --set full captures; keeps gpurun_out/ < 64 MiB.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
export CUDA_MODULE_LOADING=EAGER
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "launch list c2 rc=$?"
for c in c3 c5; do
timeout 300 python scripts/prof_once.py $c auto 1 > gpurun_out/plain_once_$c.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$c.csv python scripts/prof_once.py $c auto 1 > gpurun_out/ncu_launch_$c.log 2>&1
echo "launch list $c rc=$?"
done
timeout 300 python scripts/prof_once.py c2 auto 2 > gpurun_out/plain_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -s 1 -c 1 \
  -o gpurun_out/r01_c2_tcgemm python scripts/prof_once.py c2 auto 2 > gpurun_out/ncu_full_c2.log 2>&1
echo "ncu c2 gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hsf_pass" -s 26 -c 2 \
  -o gpurun_out/r01_c2_pass python scripts/prof_once.py c2 auto 2 > gpurun_out/ncu_full_c2p.log 2>&1
echo "ncu c2 pass rc=$?"
timeout 300 python scripts/prof_once.py c5 auto 1 > gpurun_out/plain_once_c5b.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gather|hsf_pass" -s 40 -c 3 \
  -o gpurun_out/r01_c5 python scripts/prof_once.py c5 auto 1 > gpurun_out/ncu_full_c5.log 2>&1
echo "ncu c5 rc=$?"
for f in gpurun_out/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$f" --page details > "${f%.ncu-rep}_details.txt" 2>/dev/null
  if [ $(stat -c %s "$f") -gt 15000000 ]; then rm -f "$f"; fi
done
du -sh gpurun_out
