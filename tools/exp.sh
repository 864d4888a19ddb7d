#!/bin/bash
# dev: quick per-phase timings on the GPU box (tools/quick_time.py) for a few variants
cd "$(dirname "$0")/.."
for cfg in ${CFGS:-C3}; do
  for pf in ${PFS:-l2}; do
    echo "== $cfg TC_PREFETCH=$pf"; TC_PREFETCH=$pf python tools/quick_time.py $cfg 2>&1 | tail -3
  done
done
