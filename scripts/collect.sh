#!/bin/bash
# One gpurun call's worth of round evidence: GPU suite, smoke, every config's
# bench line, the reference arm, launch lists and ncu --set full captures of
# c5's three dominant kernels. Output under gpurun_out/<tag>/ (copy the
# summaries to profiles/<tag>/ afterwards).
#   gpurun --timeout 2400 -- 'bash scripts/collect.sh r02f'
tag=${1:-collect}
out=gpurun_out/$tag
mkdir -p $out
NCU="ncu --clock-control none"
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $out/gpu_tests.log 2>&1
  tail -3 $out/gpu_tests.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
tail -1 $out/smoke.log
for c in c5 c3 c2 c1 q30-1 q32-1 q33-3; do
  timeout 400 python bench.py --config $c 2>/dev/null | tail -1 > $out/bench_$c.json
done
timeout 600 python bench.py --config c4 --steps 5 2>/dev/null | tail -1 > $out/bench_c4.json
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 > $out/bench_ref_c5.json
for c in c5 c3 c2 q33-3; do
  timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -c 400 --csv --log-file $out/launches_$c.csv python scripts/prof_once.py $c > $out/ncu_$c.log 2>&1
  python scripts/launches.py $out/launches_$c.csv > $out/launches_$c.txt 2>&1
done
# --set full of the c5 gather, half B's last pass and the T-leaf pass
# (launch ids follow launches_c5.txt: 9 = B leaf, 13 = T leaf, 14 = gather)
timeout 900 $NCU --set full --import-source on -k regex:gather_block -c 1 -o $out/c5_gather \
  python scripts/prof_once.py c5 > $out/ncu_full_gather.log 2>&1
ncu -i $out/c5_gather.ncu-rep --page details > $out/c5_gather_details.txt 2>&1
timeout 900 $NCU --set full --import-source on -k regex:hsf_jit_pass --launch-skip 5 -c 1 -o $out/c5_bleaf \
  python scripts/prof_once.py c5 > $out/ncu_full_bleaf.log 2>&1
ncu -i $out/c5_bleaf.ncu-rep --page details > $out/c5_bleaf_details.txt 2>&1
timeout 900 $NCU --set full --import-source on -k regex:hsf_jit_pass --launch-skip 9 -c 1 -o $out/c5_tleaf \
  python scripts/prof_once.py c5 > $out/ncu_full_tleaf.log 2>&1
ncu -i $out/c5_tleaf.ncu-rep --page details > $out/c5_tleaf_details.txt 2>&1
rm -f $out/*.ncu-rep
python scripts/summarize.py $out
