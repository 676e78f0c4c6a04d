#!/bin/bash
# Round refresh: full GPU suite, bench line of every config, c2 launch list +
# ncu --set full of the GEMM (the bench's dominant kernel).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r01m}
python -m paper_2502_06959_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -rf > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.log 2>&1
for c in c1 c3 c5 q30-1 q32-1 q33-3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.log 2>&1
done
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1
python scripts/summarize.py
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 300 python scripts/prof_once.py c2 auto 2 > gpurun_out/plain_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm" -s 1 -c 1 \
  -o gpurun_out/${TAG}_c2_gemm2 python scripts/prof_once.py c2 auto 2 > gpurun_out/ncu_full_c2.log 2>&1
echo "ncu gemm rc=$?"
for f in gpurun_out/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$f" --page details > "${f%.ncu-rep}_details.txt" 2>/dev/null
  rm -f "$f"
done
