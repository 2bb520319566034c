import sys, os
sys.path.insert(0, os.getcwd())
import ctypes as C, torch
from paper_1909_00899_b200 import align, workloads as W, _lib
from paper_1909_00899_b200.align import _ptr, _stream
L = _lib.load()
w = W.config1(); sch = w.scheme
r = torch.from_numpy(w.ref).cuda(); n = len(w.ref)
o3 = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(3)]
fl = torch.zeros(1, dtype=torch.uint8, device="cuda")
for lanes in (8, 16, 32, 64):
    prof = align.build_profile_arrays(w.query, sch, lanes)
    plan, pr = prof.for_kernel("scan")
    start = torch.zeros(1, dtype=torch.int64, device="cuda"); length = torch.full((1,), n, dtype=torch.int32, device="cuda")
    def fn():
        _lib.check(L.sw_db_align(C.byref(plan), _ptr(pr), 2, sch.gap_open, sch.gap_extend, prof.bias, prof.max_sub, _ptr(r), _ptr(start), _ptr(length), None, 1, None, *[_ptr(x) for x in o3], _ptr(fl), None, None, None, _stream()))
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): fn()
    e1.record(); torch.cuda.synchronize()
    print(lanes, plan.seg_len, f"{e0.elapsed_time(e1)/5:.3f} ms", [int(x) for x in o3])
