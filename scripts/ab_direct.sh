#!/bin/bash
# A/B of the direct register passes (HSF_JIT_DIRECT=0 vs default) on one box
out=${1:-gpurun_out/ab}
mkdir -p $out
for c in ${CONFIGS:-c5 c3 q32-1 q33-3}; do
  for d in 0 3 0 3; do
    HSF_JIT_DIRECT=$d timeout 300 python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | tail -1 > $out/b_${c}_$d.json
    python -c "import json,sys; d=json.load(open('$out/b_${c}_$d.json')); print('$c', 'direct=$d', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})"
  done
done
