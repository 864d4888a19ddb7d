#!/bin/bash
# dev: quick per-phase timings on the GPU box (tools/quick_time.py) for TC_EXP variants
cd "$(dirname "$0")/.."
for cfg in ${CFGS:-C3}; do
  for x in ${EXPS:-0}; do
    echo "== $cfg TC_EXP=$x"; TC_EXP=$x python tools/quick_time.py $cfg 2>&1 | tail -3 | head -2
  done
done
