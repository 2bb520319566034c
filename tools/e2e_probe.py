"""Time the pieces of the end-to-end database search (host buffers -> result)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_00899_b200 import search, workloads as W

w = W.config2()
t = time.time(); packed = search.pack(w.db, w.offsets); print(f"pack {time.time()-t:.1f}s", packed.codes.is_pinned())
eng = search.DatabaseSearch(w.scheme, coords="topk")
eng.upload(packed); eng.set_query(w.query); eng.align(); torch.cuda.synchronize()

def timed(name, fn, reps=3):
    for _ in range(1): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1)/reps:8.2f} ms (events)  {(time.perf_counter()-t0)/reps*1e3:8.2f} ms (wall)")

timed("upload", lambda: eng.upload(packed))
timed("set_query", lambda: eng.set_query(w.query))
timed("align", lambda: eng.align())
timed("upload+align", lambda: (eng.upload(packed), eng.align()))
for c in (4, 16, 32, 64, 128):
    timed(f"streamed chunks={c}", lambda: eng.search_streamed(packed, n_chunks=c))
timed("set_query+streamed16+topk", lambda: (eng.set_query(w.query), eng.search_streamed(packed, n_chunks=16), search.merge_topk(eng.topk(100), 100).cpu()))
