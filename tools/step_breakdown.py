"""Event-timed breakdown of one config-2 search step (device-resident database).

python tools/step_breakdown.py [--n-targets N] [--coords topk|all] [--frac F]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1909_00899_b200 import search, workloads as W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-targets", type=int, default=1_000_000)
    ap.add_argument("--coords", default="topk")
    ap.add_argument("--stride", type=int, default=16)
    args = ap.parse_args()
    w = W.config2(n_targets=args.n_targets)
    packed = search.pack(w.db, w.offsets)
    eng = search.DatabaseSearch(w.scheme, coords=args.coords, k=100)
    eng.SAMPLE_STRIDE = args.stride
    eng.upload(packed)
    eng.set_query(w.query)
    n = eng.dev.n
    ev = {}

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        ev.setdefault("_order", []).append(name)
        ev[name] = e

    for rep in range(3):
        ev.clear()
        mark("start")
        eng.rebuild_profile()
        mark("profile")
        order, sample = eng._sampled_order(n)
        if sample:
            eng.out["_floor"].zero_()
        eng._launch16(n, floor=bool(sample), sample=sample, order=order)
        mark("align16")
        eng._rescue(n)
        mark("rescue")
        top = eng.topk(100)
        mark("topk")
        torch.cuda.synchronize()
        names = ev["_order"]
        parts = [f"{b}={ev[a].elapsed_time(ev[b]):.3f}" for a, b in zip(names, names[1:])]
        print(f"rep {rep}: total {ev[names[0]].elapsed_time(ev[names[-1]]):.3f} ms  " + " ".join(parts),
              "floor", int(eng.out["_floor"].item()),
              "located", int((eng.out["ref_end"] != -2).sum().item()))


if __name__ == "__main__":
    main()
