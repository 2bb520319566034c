"""Timeline of the strip pipeline on config 4 (32-bit): per strip, per tile start/ready/end."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_00899_b200 import align, workloads as W
w = W.config4()
tiles = (w.ref.shape[0] + 31) // 32
nb_max = 64
buf = torch.zeros(nb_max * tiles * 4 + 4096, dtype=torch.int64, device="cuda")
os.environ["SWB_CHAIN_TRACE_PTR"] = str(buf.data_ptr())
os.environ["SWB_CHAIN_TRACE_TILES"] = str(tiles)
align.align_long(w.query, w.ref, w.scheme, width=32)
torch.cuda.synchronize()
buf.zero_()
r = align.align_long(w.query, w.ref, w.scheme, width=32)
torch.cuda.synchronize()
raw = buf.cpu().numpy()
tr = raw[: nb_max * tiles * 4].reshape(nb_max, tiles, 4)
nb = int((tr[:, 0, 0] > 0).sum())
tr = tr[:nb].astype(np.float64)
t0 = tr[:, :, 0][tr[:, :, 0] > 0].min()
tr = (tr - t0) / 1e3  # us
print("strips", nb, "result", r)
print("smid per strip:", raw[nb_max * tiles * 4: nb_max * tiles * 4 + nb].tolist())
wait = tr[:, :, 1] - tr[:, :, 0]
work = tr[:, :, 2] - tr[:, :, 1]
bp = tr[:, :, 3] - tr[:, :, 0]   # thread 31 back-pressure done, relative to tile start
print("thread-31 back-pressure done after tile start, us: median", np.median(bp[:, 10:]), "strip0", np.median(bp[0, 10:]))
print("per-tile work us: median", np.median(work), "p90", np.percentile(work, 90))
print("per-tile wait us: median", np.median(wait), "p90", np.percentile(wait, 90))
for b in range(nb):
    if b < 3 or b == nb - 1: print(f"strip {b:2d} start {tr[b,0,0]:9.1f} end {tr[b,-1,2]:9.1f} work {work[b].sum()/1e3:7.2f} ms wait {wait[b].sum()/1e3:7.2f} ms")
print("strip0 work every 100 tiles (us):", np.round(work[0, ::100], 1).tolist())
print("strip0 bp every 100 tiles (us):", np.round(bp[0, ::100], 1).tolist())
print("strip1 work every 100 tiles (us):", np.round(work[1, ::100], 1).tolist())
print("strip1 wait per tile 0..40 (us):", np.round(wait[1, :40], 1).tolist())
print("strip0 bp per tile 0..40 (us):", np.round(bp[0, :40], 1).tolist())
print("tile 100 start per strip:", np.round(tr[:, 100, 0], 1))
print("strip0 tiles 0..12 [start,ready,end,bp]:", np.round(tr[0, :12], 1).tolist())
print("strip0 tiles 1000..1004:", np.round(tr[0, 1000:1004], 1).tolist())
print("strip1 tiles 1000..1004:", np.round(tr[1, 1000:1004], 1).tolist())
np.save(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "chain_trace.npy"), tr)
