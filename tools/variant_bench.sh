#!/bin/bash
# Time the config-2 kernel for each library variant under build/var_*/ (and the in-tree one).
cd "$(dirname "$0")/.."
echo "== in-tree"; python tools/prof_db.py --n-targets 1000000 --reps 3 | tail -2
for so in _variants/*/libswscan_b200.so; do
  echo "== $so"; SWB_LIB_PATH=$PWD/$so python tools/prof_db.py --n-targets 1000000 --reps 3 | tail -2
done
