cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for c in c2 c1 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  HSF_NO_GRAPH=1 timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${c}_nograph.log 2>&1
done
python scripts/summarize.py
