"""Minimal driver for profiling the config-2 database kernel under ncu.

python tools/prof_db.py [--n-targets N] [--reps R] [--lanes P] [--kernel scan|lazyf]
Runs R launches of the 16-bit striped kernel (no rescue, no top-k) and prints
the event-timed GCUPS of each launch.
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-targets", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--kernel", default="scan")
    ap.add_argument("--floor-topk", type=int, default=0,
                    help="after one full run, use the k-th best score as the coordinate floor")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_1909_00899_b200 import align, workloads as W

    w = W.config2(n_targets=args.n_targets)
    prof = align.build_profile_arrays(w.query, w.scheme, args.lanes)
    tgt = torch.from_numpy(w.db).cuda()
    start = torch.from_numpy(w.offsets[:-1].copy()).cuda()
    length = torch.from_numpy(np.diff(w.offsets).astype(np.int32)).cuda()
    order = torch.from_numpy(np.argsort(-np.diff(w.offsets), kind="stable").astype(np.int32)).cuda()
    cells = w.cells
    print("plan", prof.plan16)
    floor = None
    if args.floor_topk:
        o = align.db_align(prof, tgt, start, length, order, args.kernel, rescue=False)
        floor = torch.topk(o["score"], args.floor_topk).values.min().reshape(1).to(torch.int32)
        print("coordinate floor", int(floor.item()))
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        align.db_align(prof, tgt, start, length, order, args.kernel, rescue=False,
                       coord_floor=floor)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{ms:.3f} ms  {cells / ms / 1e6:.1f} GCUPS")


if __name__ == "__main__":
    main()
