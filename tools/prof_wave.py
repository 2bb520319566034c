"""Driver for profiling the wavefront strip pipeline under ncu: one config-5 long pair
(or a slice: --m/--n) through sw_align_long(kernel=wavefront), event-timed."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1909_00899_b200 import align, workloads as W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--kernel", default="wavefront")
    args = ap.parse_args()
    w = W.config5()
    q = w.query[: args.m] if args.m else w.query
    r = w.ref[: args.n] if args.n else w.ref
    qd, rd = torch.from_numpy(q).cuda(), torch.from_numpy(r).cuda()
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = align.align_long(q, r, w.scheme, kernel=args.kernel, query_dev=qd, ref_dev=rd)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{args.kernel} {q.shape[0]}x{r.shape[0]}: {ms:.3f} ms "
              f"{q.shape[0] * r.shape[0] / ms / 1e6:.1f} GCUPS {res}")


if __name__ == "__main__":
    main()
