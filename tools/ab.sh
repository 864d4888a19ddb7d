#!/bin/bash
# dev: same-box A/B of library variants (build/<name>/libtriadcensus.so, built by
# tools/build_variant.sh) against the in-tree library, interleaved, on CFGS.
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for cfg in ${CFGS:-C3}; do
    echo "== $cfg base"; python tools/quick_time.py $cfg 2>&1 | tail -3 | head -2
    for v in ${VARIANTS}; do
      echo "== $cfg $v"; TC_LIB_VARIANT=build/$v/libtriadcensus.so python tools/quick_time.py $cfg 2>&1 | tail -3 | head -2
    done
  done
done
