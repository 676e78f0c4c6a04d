#!/bin/bash
# One GPU round trip: parity tests, smoke, benches of the given configs.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_check.sh [configs...]'
# (q-configs = Table II-shaped QAOA, benched with --standard for T/J)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CFGS=${@:-c2 c1 c3 c5 c4}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 -rf > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
for c in $CFGS; do
  extra=""; [ "$c" != "c2" ] && extra="--no-cpu-baseline"
  case $c in q*) extra="$extra --standard";; esac
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 $extra > gpurun_out/bench_$c.log 2>&1
  echo "bench $c rc=$?" >> gpurun_out/bench_$c.log
done
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log
for c in $CFGS; do tail -2 gpurun_out/bench_$c.log | cut -c1-300; done
