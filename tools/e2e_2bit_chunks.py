"""Config-3 end-to-end step from 2-bit packed pinned input at several chunk counts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1909_00899_b200 import workloads as W
from paper_1909_00899_b200.align import PairsBatch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
w = W.config3(n_pairs=n)
b0 = PairsBatch(w.scheme)
for packed in (True, False):
    host = b0.pin_host(w.flat_q, w.q_off, w.flat_r, w.r_off, packed2bit=packed)
    for nc in (4, 8, 16, 32, 64):
        b = PairsBatch(w.scheme, coords=False)
        b.prepare_host(host, n_chunks=nc)
        b.run_host(host)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            b.run_host(host)
            torch.cuda.current_stream().synchronize()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"packed2bit={packed} chunks={nc}: {ms:.2f} ms, {w.cells / ms / 1e6:.1f} GCUPS, h2d {b.h2d_bytes / 1e6:.0f} MB")
    del host
