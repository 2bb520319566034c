"""Sweep the wavefront strip tile shape (rows per lane L x columns per step KC) on
configs 1, 4 and 5 (event-timed sw_align_long, resident inputs, workspace reused).

python tools/wave_sweep.py [--configs 1,4,5] [--reps R]
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1909_00899_b200 import workloads as W  # noqa: E402

import bench_configs as B  # noqa: E402  (tools/ is on sys.path when run as a script)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,4,5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--L", default="1,2,4,8")
    ap.add_argument("--KC", default="1,2,4,8")
    args = ap.parse_args()
    ws = {"1": W.config1, "4": W.config4, "5": W.config5}
    for c in args.configs.split(","):
        w = ws[c]()
        for L in args.L.split(","):
            for kc in args.KC.split(","):
                os.environ["SWB_WAVE_L"], os.environ["SWB_WAVE_KC"] = L, kc
                B.long_pair(f"config{c}[L={L},KC={kc}]", w, args.reps, kernel="wavefront")
    os.environ.pop("SWB_WAVE_L", None)
    os.environ.pop("SWB_WAVE_KC", None)


if __name__ == "__main__":
    main()
