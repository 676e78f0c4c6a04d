#!/bin/bash
# A/B of the heavy passes' min CTAs per SM and the shared-memory carveout on one box
out=${1:-gpurun_out/ab_minb}
mkdir -p $out
for c in ${CONFIGS:-c5 q32-1 q33-3 c3}; do
  for rep in 1 2; do
    for v in "4:" "5:" "5:100" "4:100"; do
      mb=${v%%:*}; co=${v##*:}
      if [ -n "$co" ]; then export HSF_JIT_CARVEOUT=$co; else unset HSF_JIT_CARVEOUT; fi
      HSF_JIT_HEAVY_MINB=$mb timeout 300 python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | tail -1 > $out/b_${c}_${mb}_${co}.json
      python -c "import json,sys; d=json.load(open('$out/b_${c}_${mb}_${co}.json')); print('$c', 'minb=$mb carveout=$co', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})"
    done
  done
done
