"""Bisect a strip-pipeline mismatch: same pair, both widths, forced strip lengths."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

TRIAL = int(sys.argv[1]) if len(sys.argv) > 1 else 2


def inputs(trial):
    rng = np.random.default_rng(0x10C)
    for t in range(trial + 1):
        k = int(rng.integers(2, 21)); mat = rng.integers(-5, 6, (k, k))
        go = int(rng.integers(1, 12)); ge = int(rng.integers(1, go + 1))
        m = int(rng.integers(1, 9000)); n = int(rng.integers(1, 3000))
        q = rng.integers(0, k, m).astype(np.uint8); r = rng.integers(0, k, n).astype(np.uint8)
        if t % 2:
            blk = q[: min(m, n)]; r[: blk.shape[0]] = blk
    return q, r, mat, go, ge


if __name__ == "__main__":
    if os.environ.get("SWB_CHILD"):
        from oracle import oracle as O
        from paper_1909_00899_b200 import align
        from paper_1909_00899_b200.scoring import ScoringScheme
        q, r, mat, go, ge = inputs(TRIAL)
        sch = ScoringScheme.from_array(mat, go, ge)
        want = O.scalar(q, r, mat, go, ge)
        for w in (16, 32):
            g = align.align_long(q, r, sch, width=w)
            print(os.environ.get("SWB_CHAIN_L", "auto"), "width", w, (g["score"], g["ref_end"], g["query_end"]), "oracle", want)
    else:
        for L in ("auto", "4", "8", "16", "32"):
            env = dict(os.environ, SWB_CHILD="1")
            if L != "auto":
                env["SWB_CHAIN_L"] = L
            subprocess.run([sys.executable, __file__, str(TRIAL)], env=env)
