#!/bin/bash
# A/B of one environment knob on one box: scripts/ab_env.sh <out> <VAR> <a> <b> [configs]
out=$1; var=$2; a=$3; b=$4; shift 4
mkdir -p $out
for c in ${@:-c5 q32-1 q33-3}; do
  for d in $a $b $a $b; do
    env $var=$d timeout 300 python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | tail -1 > $out/b_${c}_${var}_$d.json
    python -c "import json,sys; d=json.load(open('$out/b_${c}_${var}_$d.json')); print('$c', '$var=$d', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})"
  done
done
