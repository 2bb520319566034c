"""Profile driver: config-3 pairs kernel, score-only (the metric's launch), on the
first 2^20 pairs through PairsBatch (16-bit launch + device-counted rescue)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1909_00899_b200 import align, workloads as W

w = W.config3(n_pairs=1 << 20)
b = align.PairsBatch(w.scheme, coords=os.environ.get("C3_COORDS") == "1",
                     lanes=int(os.environ.get("C3_LANES", "0")))
b.upload(w.flat_q, w.q_off, w.flat_r, w.r_off)
b.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
o = b.run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"{ms:.3f} ms, {w.cells / ms / 1e6:.1f} GCUPS, score sum {int(o['score'][:w.n_pairs].sum())}")
