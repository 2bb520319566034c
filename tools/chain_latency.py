"""Strip-pipeline per-column latency: ns per reference column for one strip alone
(m = 32 * L) and for a full pipeline of `nb` strips, at each strip height L.

python tools/chain_latency.py [--n 200000] [--nb 512]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1909_00899_b200 import align, workloads as W


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200000)
    ap.add_argument("--nb", type=int, default=512)
    ap.add_argument("--Ls", default="4,8,16,32")
    ap.add_argument("--m", type=int, default=0, help="fixed query length (nb = m / 32L)")
    ap.add_argument("--kernel", default="scan", choices=["scan", "wavefront"])
    args = ap.parse_args()
    rng = np.random.default_rng(7)
    w = W.config5()
    ref = w.ref[: args.n].copy()
    for L in (int(x) for x in args.Ls.split(",")):
        os.environ["SWB_WAVE_L" if args.kernel == "wavefront" else "SWB_CHAIN_L"] = str(L)
        for nb in ((1, args.nb) if not args.m else (1, max(1, args.m // (32 * L)))):
            q = w.query[: 32 * L * nb].copy()
            if q.shape[0] < 32 * L * nb:
                q = rng.integers(0, 4, 32 * L * nb).astype(np.uint8)
            align.align_long(q, ref, w.scheme, width=32, kernel=args.kernel)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = align.align_long(q, ref, w.scheme, width=32, kernel=args.kernel)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            cols = ref.shape[0] + 32 * (nb - 1)
            print(f"L={L:2d} nb={nb:4d} score={r['score']:6d} {ms:8.2f} ms  "
                  f"{ms * 1e6 / cols:6.1f} ns/col  {ms * 1e6 / cols * 1.965:6.0f} cyc/col  "
                  f"{q.shape[0] * ref.shape[0] / ms / 1e6:7.1f} GCUPS", flush=True)
    os.environ.pop("SWB_CHAIN_L", None)
    os.environ.pop("SWB_WAVE_L", None)


if __name__ == "__main__":
    main()
