"""One strip only (m = 128, 32-bit, L = 4): no producer/consumer; per-column time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_00899_b200 import align, workloads as W
w = W.config4()
q = w.query[:128]
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = align.align_long(q, w.ref, w.scheme, width=32); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print("single strip", r, f"{ms:.2f} ms = {ms * 1e6 / w.ref.shape[0]:.0f} ns/column")
