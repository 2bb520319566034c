"""Per-configuration device throughput (GCUPS), inputs resident in HBM, event-timed.

python tools/bench_configs.py [--configs 1,3,4,5] [--c3-pairs N] [--reps R]

Config 2 (the headline) is bench.py. Prints one JSON line per (config, kernel);
the long-pair path (configs 4/5 in 32-bit) is the strip pipeline.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1909_00899_b200 import _lib, align, workloads as W
from paper_1909_00899_b200.align import _ptr, _stream


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def emit(**kw):
    print(json.dumps(kw), flush=True)


def single_pair(name, w, kernels, lanes, reps, width=16):
    """One pair through the warp kernel (sw_db_align with n = 1), device-resident."""
    L = _lib.load()
    prof = align.build_profile_arrays(w.query, w.scheme, lanes)
    tgt = torch.from_numpy(w.ref).cuda()
    start = torch.zeros(1, dtype=torch.int64, device="cuda")
    length = torch.full((1,), w.ref.shape[0], dtype=torch.int32, device="cuda")
    out = {k: torch.empty(1, dtype=torch.int32, device="cuda") for k in ("s", "r", "q")}
    fl = torch.empty(1, dtype=torch.uint8, device="cuda")
    sch = w.scheme
    for kern in kernels:
        kid = _lib.KERNEL_IDS[kern]

        def run():
            _lib.check(L.sw_db_align(C.byref(prof.plan16), _ptr(prof.prof16), kid, sch.gap_open,
                                     sch.gap_extend, prof.bias, prof.max_sub, _ptr(tgt),
                                     _ptr(start), _ptr(length), None, 1, None, _ptr(out["s"]),
                                     _ptr(out["r"]), _ptr(out["q"]), _ptr(fl), None, None, None, _stream()))

        ms = timed(run, reps)
        emit(config=name, kernel=kern, width=16, lanes=prof.plan16.lanes, seg_len=prof.plan16.seg_len,
             ms=round(ms, 4), gcups=round(w.cells / ms / 1e6, 3), score=int(out["s"].item()),
             ref_end=int(out["r"].item()), query_end=int(out["q"].item()), path="warp kernel")


def long_pair(name, w, reps, width=32, kernel="scan"):
    L = _lib.load()
    q = torch.from_numpy(w.query).cuda()
    r = torch.from_numpy(w.ref).cuda()
    sub = torch.from_numpy(w.scheme.as_array()).cuda()
    m, n = int(q.numel()), int(r.numel())
    nbytes = int(L.sw_long_workspace_bytes(m, n, w.scheme.n_symbols, width))
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = torch.empty(3, dtype=torch.int32, device="cuda")
    fl = torch.empty(1, dtype=torch.uint8, device="cuda")
    sch = w.scheme

    def run():
        _lib.check(L.sw_align_long(width, _lib.KERNEL_IDS[kernel], _ptr(q), m, _ptr(r), n,
                                   _ptr(sub), sch.n_symbols,
                                   sch.gap_open, sch.gap_extend, sch.bias, sch.max_score, _ptr(ws),
                                   nbytes, C.c_void_p(out.data_ptr()),
                                   C.c_void_p(out.data_ptr() + 4), C.c_void_p(out.data_ptr() + 8),
                                   _ptr(fl), _stream()))

    ms = timed(run, reps)
    o = out.cpu().tolist()
    emit(config=name, kernel=kernel, width=32 if kernel == "wavefront" else width,
         ms=round(ms, 3), gcups=round(w.cells / ms / 1e6, 3), score=o[0], ref_end=o[1],
         query_end=o[2], path="strip pipeline (sw_align_long)")


def pairs(name, w, reps, kernels=("scan", "lazyf"), lanes=0, coords=True):
    L = _lib.load()
    n = w.n_pairs
    qlen = np.diff(w.q_off).astype(np.int32)
    tlen = np.diff(w.r_off).astype(np.int32)
    dev = {"q": torch.from_numpy(w.flat_q).cuda(), "qs": torch.from_numpy(w.q_off[:-1].copy()).cuda(),
           "ql": torch.from_numpy(qlen).cuda(), "t": torch.from_numpy(w.flat_r).cuda(),
           "ts": torch.from_numpy(w.r_off[:-1].copy()).cuda(), "tl": torch.from_numpy(tlen).cuda()}
    sub = torch.from_numpy(w.scheme.as_array()).cuda()
    out = {k: torch.empty(n, dtype=torch.int32, device="cuda") for k in ("s", "r", "q")}
    fl = torch.empty(n, dtype=torch.uint8, device="cuda")
    sch = w.scheme
    for kern in kernels:
        kid = _lib.KERNEL_IDS[kern]

        def run():
            _lib.check(L.sw_pairs_align(16, lanes, kid, _ptr(dev["q"]), _ptr(dev["qs"]), _ptr(dev["ql"]),
                                        _ptr(dev["t"]), _ptr(dev["ts"]), _ptr(dev["tl"]), None, n,
                                        None, int(qlen.min()), int(qlen.max()), _ptr(sub),
                                        sch.n_symbols, sch.gap_open, sch.gap_extend, sch.bias,
                                        sch.max_score, None, None, None, None, _ptr(out["s"]),
                                        _ptr(out["r"]) if coords else None,
                                        _ptr(out["q"]) if coords else None, _ptr(fl), None, None,
                                        _stream()))

        ms = timed(run, reps)
        emit(config=name, kernel=kern, width=16, pairs=n, lanes=lanes, ms=round(ms, 3),
             gcups=round(w.cells / ms / 1e6, 3), coords=coords,
             path="pairs kernel (per-pair profiles)")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5")
    ap.add_argument("--c3-pairs", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--c3-lanes", default="0")
    args = ap.parse_args()
    cfgs = {int(x) for x in args.configs.split(",")}
    if 1 in cfgs:
        w = W.config1()
        single_pair("config1", w, ("scan", "lazyf", "lazyf-noexit"), 0, args.reps * 10)
        for ln in (16, 32, 64):
            single_pair("config1", w, ("scan", "lazyf"), ln, args.reps * 10)
        long_pair("config1", w, args.reps * 10, kernel="wavefront")
    if 3 in cfgs:
        w3 = W.config3(n_pairs=args.c3_pairs)
        for ln in (int(x) for x in args.c3_lanes.split(",")):
            pairs(f"config3[{args.c3_pairs} pairs]", w3, args.reps, lanes=ln,
                  kernels=("scan", "lazyf") if ln == 0 else ("scan",))
            pairs(f"config3[{args.c3_pairs} pairs]", w3, args.reps, lanes=ln,
                  kernels=("scan",), coords=False)
    if 4 in cfgs:
        w = W.config4()
        single_pair("config4", w, ("scan", "lazyf", "lazyf-noexit"), 64, args.reps)
        long_pair("config4", w, args.reps, width=32)
        long_pair("config4", w, args.reps, kernel="wavefront")
    if 5 in cfgs:
        w5 = W.config5()
        long_pair("config5", w5, max(1, args.reps // 2), width=32)
        long_pair("config5", w5, args.reps, kernel="wavefront")


if __name__ == "__main__":
    main()
