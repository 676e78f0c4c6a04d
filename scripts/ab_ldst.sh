#!/bin/bash
# A/B of the generated passes' state load / store cache operators (HSF_JIT_LDST = 10 * ld + st) on one box
out=${1:-gpurun_out/ab_ldst}
mkdir -p $out
for c in ${CONFIGS:-c5 q33-3}; do
  for rep in 1 2; do
    for v in ${MODES:-0 2 1 20 22 10 12}; do
      HSF_JIT_LDST=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | tail -1 > $out/b_${c}_$v.json
      python -c "import json,sys; d=json.load(open('$out/b_${c}_$v.json')); print('$c', 'ldst=$v', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})"
    done
  done
done
