#!/bin/bash
# A/B of the config-3 pairs kernel only: in-tree library against vt/<name>/libswscan_b200.so
cd "$(dirname "$0")/.."
for so in "" vt/*/libswscan_b200.so; do
  echo "== ${so:-in-tree}"
  if [ -n "$so" ]; then export SWB_LIB_PATH=$PWD/$so; else unset SWB_LIB_PATH; fi
  python tools/bench_configs.py --configs 3 --c3-pairs 16777216 --reps 3 | grep -v lazyf | cut -c1-140
done
