#!/bin/bash
# A/B wavefront variants (vt/<name>/libswscan_b200.so) on config 5 (and 4, 1).
cd "$(dirname "$0")/.."
for so in "" vt/*/libswscan_b200.so; do
  echo "== ${so:-in-tree}"
  if [ -n "$so" ]; then export SWB_LIB_PATH=$PWD/$so; else unset SWB_LIB_PATH; fi
  python tools/bench_configs.py --configs 1,4,5 --reps 3 | grep -E "wavefront|strip pipeline" | cut -c1-110
done
