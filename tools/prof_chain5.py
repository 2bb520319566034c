"""Profile driver: config 5 through the strip pipeline (32-bit), one launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_00899_b200 import align, workloads as W
w = W.config5()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); r = align.align_long(w.query, w.ref, w.scheme, width=32); e1.record(); torch.cuda.synchronize()
print(r, f"{e0.elapsed_time(e1):.1f} ms")
