"""Start coordinates (beyond the reference): the oracle's
anchored reverse DP (swo_start_coords) against an exhaustive search over every
candidate start on small pairs, including the reference-pinned end cells of
tests/golden/coords_small.npz (from the reference's own DP matrices)."""

from __future__ import annotations

import numpy as np

from helpers import golden, mm_matrix

NEG = -(1 << 40)


def anchored_both(q, r, sub, go, ge, i0, q0, i1, q1):
    """Best score of an alignment whose first aligned pair is (i0, q0) and whose
    last aligned pair is (i1, q1) (reference index i, query index q), Gotoh gaps
    (open go counts the first gap position, extend ge each further one)."""
    n, m = i1 - i0 + 1, q1 - q0 + 1
    H = np.full((n, m), NEG, dtype=np.int64)
    E = np.full((n, m), NEG, dtype=np.int64)  # gap along the reference (i)
    F = np.full((n, m), NEG, dtype=np.int64)  # gap along the query (q)
    U = np.full((n, m), NEG, dtype=np.int64)  # diagonal (aligned pair) entry
    for a in range(n):
        for b in range(m):
            s = int(sub[r[i0 + a], q[q0 + b]])
            if a == 0 and b == 0:
                U[a, b] = s
            elif a > 0 and b > 0 and H[a - 1, b - 1] > NEG // 2:
                U[a, b] = H[a - 1, b - 1] + s
            if a > 0:
                E[a, b] = max(E[a - 1, b] - ge, H[a - 1, b] - go)
            if b > 0:
                F[a, b] = max(F[a, b - 1] - ge, H[a, b - 1] - go)
            H[a, b] = max(U[a, b], E[a, b], F[a, b])
    return int(U[n - 1, m - 1])


def brute_start(q, r, sub, go, ge, score, re_, qe):
    # first in (ref_end - i0 ascending, query_end - q0 ascending) order
    for i0 in range(re_, -1, -1):
        for q0 in range(qe, -1, -1):
            if anchored_both(q, r, sub, go, ge, i0, q0, re_, qe) == score:
                return i0, q0
    return None


def test_start_coords_exhaustive_random(oracle):
    rng = np.random.default_rng(0x57A7)
    for trial in range(120):
        k = int(rng.integers(2, 6))
        sub = rng.integers(-4, 5, (k, k))
        np.fill_diagonal(sub, np.abs(np.diag(sub)) + 1)
        go = int(rng.integers(1, 6))
        ge = int(rng.integers(1, go + 1))
        q = rng.integers(0, k, int(rng.integers(1, 11))).astype(np.uint8)
        r = rng.integers(0, k, int(rng.integers(1, 11))).astype(np.uint8)
        score, re_, qe = oracle.scalar(q, r, sub, go, ge)
        got = oracle.start_coords(q, r, sub, go, ge, score, re_, qe)
        if score == 0:
            assert got == (-1, -1)
            continue
        assert got == brute_start(q, r, sub, go, ge, score, re_, qe), (trial, q, r, sub, go, ge)


def test_start_coords_reference_pinned_ends(oracle):
    """End cells pinned by the reference's own H matrices (coords_small.npz);
    starts checked exhaustively on the short ones, and consistency on all."""
    g = golden("coords_small.npz")
    q_off, r_off = g["q_off"], g["r_off"]
    checked = 0
    for t in range(q_off.shape[0] - 1):
        q = g["flat_q"][q_off[t]:q_off[t + 1]]
        r = g["flat_r"][r_off[t]:r_off[t + 1]]
        sub = mm_matrix(int(g["match"][t]), int(g["mismatch"][t]), 4)
        go, ge = int(g["go"][t]), int(g["ge"][t])
        score, re_, qe = int(g["score"][t]), int(g["ref_end"][t]), int(g["query_end"][t])
        rs, qs = oracle.start_coords(q, r, sub, go, ge, score, re_, qe)
        if score == 0:
            assert (rs, qs) == (-1, -1)
            continue
        assert 0 <= rs <= re_ and 0 <= qs <= qe
        # the sub-alignment [rs..re] x [qs..qe] scores exactly the best local score
        assert oracle.scalar(q[qs:qe + 1], r[rs:re_ + 1], sub, go, ge)[0] == score
        if (re_ - rs + 1) * (qe - qs + 1) <= 400 and checked < 60:
            assert (rs, qs) == brute_start(q, r, sub, go, ge, score, re_, qe), t
            checked += 1
    assert checked > 20


def test_batch_starts_matches_single(oracle):
    rng = np.random.default_rng(5)
    sub = mm_matrix(2, -3, 4)
    n = 50
    ql = rng.integers(1, 60, n)
    tl = rng.integers(1, 80, n)
    q_off = np.concatenate([[0], np.cumsum(ql)]).astype(np.int64)
    r_off = np.concatenate([[0], np.cumsum(tl)]).astype(np.int64)
    fq = rng.integers(0, 4, q_off[-1]).astype(np.uint8)
    fr = rng.integers(0, 4, r_off[-1]).astype(np.uint8)
    s, re_, qe = oracle.batch_scalar(fq, q_off, fr, r_off, sub=sub, go=5, ge=2)
    rs, qs = oracle.batch_starts(fq, q_off, fr, r_off, sub, 5, 2, s, re_, qe)
    for t in range(n):
        want = oracle.start_coords(fq[q_off[t]:q_off[t + 1]], fr[r_off[t]:r_off[t + 1]], sub, 5, 2,
                                   int(s[t]), int(re_[t]), int(qe[t]))
        assert (rs[t], qs[t]) == want
