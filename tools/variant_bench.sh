#!/bin/bash
# A/B the in-tree library against variants built into vt/<name>/libswscan_b200.so
# (make -C paper_1909_00899_b200/csrc VARIANT_FLAGS=... OUT=../../vt/<name>/libswscan_b200.so
#  BUILD=../../build/var_<name>): config-2 kernel (auto plan and 16 stripes) and config-3 pairs, same box.
cd "$(dirname "$0")/.."
for so in "" vt/*/libswscan_b200.so; do
  echo "== ${so:-in-tree}"
  if [ -n "$so" ]; then export SWB_LIB_PATH=$PWD/$so; else unset SWB_LIB_PATH; fi
  python tools/prof_db.py --n-targets 1000000 --reps 3 --floor-topk 100 | tail -2
  echo "-- 16 stripes (SWB_PLAN_MAX_L=32)"
  SWB_PLAN_MAX_L=32 python tools/prof_db.py --n-targets 1000000 --reps 3 --floor-topk 100 | tail -2
  python tools/bench_configs.py --configs 3 --c3-pairs 16777216 --reps 3 | grep -v lazyf | cut -c1-140
done
