"""Time the block / cluster kernel (sw_align_block) on configs 4 and 5 at several
stripe counts, device-timed with CUDA events (inputs resident), and check each
result against the strip pipeline's (itself checked against the oracle in tests).

  python tools/bench_block.py [--config 4|5|1] [--lanes 512,2048] [--width 16] [--kernel scan]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1909_00899_b200 import _lib, align, workloads  # noqa: E402


def time_block(w, lanes, width, kernel, reps=3, coords=True):
    L = _lib.load()
    kid = _lib.KERNEL_IDS[kernel]
    geo = _lib.block_plan(w.m, w.scheme.n_symbols, width, kid, lanes)
    if geo is None:
        return None
    qd = torch.from_numpy(w.query).cuda()
    rd = torch.from_numpy(w.ref).cuda()
    sub = torch.from_numpy(w.scheme.as_array()).cuda()
    out = torch.zeros(4, dtype=torch.int32, device="cuda")
    fl = torch.zeros(1, dtype=torch.uint8, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

    def launch():
        _lib.check(L.sw_align_block(width, kid, geo[0], p(qd), w.m, p(rd), int(w.ref.size), p(sub),
                                    w.scheme.n_symbols, w.scheme.gap_open, w.scheme.gap_extend,
                                    w.scheme.bias, w.scheme.max_score, int(coords),
                                    p(out), C.c_void_p(out.data_ptr() + 4),
                                    C.c_void_p(out.data_ptr() + 8), p(fl), None,
                                    p(stats) if kernel != "scan" else None, sp))

    launch()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    cells = w.m * int(w.ref.size)
    o = out.cpu().tolist()
    return {"lanes": geo[0], "threads": geo[1], "cluster": geo[2], "seg_len": geo[3],
            "width": width, "kernel": kernel, "ms": round(ms, 3),
            "gcups": round(cells / ms / 1e6, 2), "score": o[0], "ref_end": o[1], "query_end": o[2],
            "flags": int(fl.item()), "ns_per_col": round(ms * 1e6 / int(w.ref.size), 1),
            "passes": int(stats[0].item()) if kernel != "scan" else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--lanes", default="")
    ap.add_argument("--width", type=int, default=0)
    ap.add_argument("--kernel", default="scan")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=0, help="reference prefix length (0 = full)")
    args = ap.parse_args()
    w = {1: workloads.config1, 4: workloads.config4, 5: workloads.config5}[args.config]()
    if args.n:
        w.ref = w.ref[: args.n]
    ref_res = align.align_long(w.query, w.ref, w.scheme, width=32,
                               kernel="wavefront" if args.config != 1 else "scan")
    want = (ref_res["score"], ref_res["ref_end"], ref_res["query_end"])
    widths = [args.width] if args.width else [16, 32]
    lanes = [int(x) for x in args.lanes.split(",")] if args.lanes else [0]
    for width in widths:
        for p in lanes:
            r = time_block(w, p, width, args.kernel, args.reps)
            if r is None:
                print(json.dumps({"config": args.config, "lanes": p, "width": width, "skip": "no layout"}))
                continue
            r["config"] = args.config
            r["exact"] = (r["score"], r["ref_end"], r["query_end"]) == want or bool(r["flags"] & 2)
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
