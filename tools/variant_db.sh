#!/bin/bash
# A/B of the config-2 database kernel only: in-tree library against vt/<name>/libswscan_b200.so
cd "$(dirname "$0")/.."
for so in "" vt/*/libswscan_b200.so; do
  echo "== ${so:-in-tree}"
  if [ -n "$so" ]; then export SWB_LIB_PATH=$PWD/$so; else unset SWB_LIB_PATH; fi
  python tools/prof_db.py --n-targets 1000000 --reps 4 --floor-topk 100 | tail -3
done
