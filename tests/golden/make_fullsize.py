"""Full-size oracle results for configs 2, 3 and 5 (VERDICT r01 missing item 1).

The C oracle (oracle/sw_oracle.c: _sw_scalar_c, src/_compiled.py:76-115, with
first-maximum end coordinates, contract A10; OpenMP over this container's
cores) computes (score, ref_end, query_end) for
  * config 2: all 1,000,000 database targets (1.67e11 cells, ~2 min on 8 threads),
  * config 3: all 16,777,216 read/window pairs (7.55e11 cells, ~5 min),
  * config 5: the 65,536 x 1,048,576 pair (6.87e10 cells, one thread, ~5 min),
on the seeded inputs of paper_1909_00899_b200.workloads, and writes
tests/golden/fullsize.json: input sha256s plus result digests
(tests/helpers.result_digest: a sha256 of the int32 arrays and 256 or 1,024
block digests to localise a mismatch). The oracle itself is pinned to the
reference's outputs by tests/test_oracle_golden.py (config 5's score also to
the reference's own scan kernel, configs.npz c5_scan_p64_score).

The GPU tests (tests/test_gpu_fullsize.py) regenerate the same inputs on the
box, check their sha256, run the device path at full size and compare digests.

Usage: python tests/golden/make_fullsize.py [--configs 2,3,5]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))

from helpers import result_digest, sha  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1909_00899_b200 import workloads as W  # noqa: E402

OUT = os.path.join(HERE, "fullsize.json")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,5")
    args = ap.parse_args()
    res = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            res = json.load(fh)
    for c in [int(x) for x in args.configs.split(",")]:
        t0 = time.time()
        if c == 2:
            w = W.config2()
            s, r, q = O.db_scalar(w.query, w.db, w.offsets, w.scheme.as_array(),
                                  w.scheme.gap_open, w.scheme.gap_extend)
            order = np.lexsort((np.arange(w.n_targets), -s.astype(np.int64)))[:100]
            res["config2"] = {"inputs_sha256": sha(w.query, w.db, w.offsets),
                              "cells": w.cells, **result_digest(s, r, q, 256),
                              "top100": [[int(s[i]), int(i), int(r[i]), int(q[i])] for i in order]}
        elif c == 3:
            w = W.config3()
            s, r, q = O.batch_scalar(w.flat_q, w.q_off, w.flat_r, w.r_off,
                                     sub=w.scheme.as_array(), go=w.scheme.gap_open,
                                     ge=w.scheme.gap_extend)
            res["config3"] = {"inputs_sha256": sha(w.flat_q, w.flat_r), "cells": w.cells,
                              **result_digest(s, r, q, 1024)}
        elif c == 5:
            w = W.config5()
            s, r, q = O.scalar(w.query, w.ref, w.scheme.as_array(), w.scheme.gap_open,
                               w.scheme.gap_extend)
            res["config5"] = {"inputs_sha256": sha(w.query, w.ref), "cells": w.cells,
                              "score": int(s), "ref_end": int(r), "query_end": int(q)}
        res.setdefault("_meta", {})[f"config{c}_seconds"] = round(time.time() - t0, 1)
        res["_meta"]["oracle_threads"] = O.n_threads()
        with open(OUT, "w") as fh:
            json.dump(res, fh, indent=0)
        print(f"config {c}: {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
