#!/bin/bash
# Relaxed vs strict gate passes on the bench circuits (digest must match).
# usage: bash tools/bench_matrix.sh [circuits...]
circs=${@:-qft qaoa supremacy}
for c in $circs; do
  for a in "" "--strict-passes"; do
    timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --circuit $c $a 2>&1 | tail -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $a', round(d['value'],1), {k: round(v,4) for k,v in d['phases_s'].items()}, d['gate_passes'], d['replays'], d['digest'])"
  done
done
