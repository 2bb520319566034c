"""Every exact-L scan instance of the striped kernel against the scalar oracle.

The database kernels are compiled per (threads, segment length, gap-extend
specialisation); instances with a compile-time gap extend use the 3-input
deferred correction (FUSE3: all words for segments up to 32 words, the first
words of longer segments).  This sweep launches each of them -- every segment
length 1..64 at every group width that has instances, gap extend 1, 2 and 3
(the runtime-ge instances) -- on targets that contain planted, mutated pieces
of the query (long diagonals, gaps, lane and word boundaries crossed), and
compares scores and end coordinates with `_sw_scalar_c`'s restatement
(src/_compiled.py:76-115).  Exact equality.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def A():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_00899_b200 import align

    return align


def _targets(rng, q, k, n_targets=24):
    """Targets with a mutated slice of the query planted in random background."""
    seqs = []
    m = q.shape[0]
    for i in range(n_targets):
        bg = rng.integers(0, k, int(rng.integers(1, 160))).astype(np.uint8)
        if i % 6 == 5 or m < 2:
            seqs.append(bg)
            continue
        a = int(rng.integers(0, m))
        b = int(rng.integers(a + 1, min(m, a + 260) + 1))
        piece = q[a:b].copy()
        sub = rng.random(piece.shape[0]) < 0.06
        piece[sub] = rng.integers(0, k, int(sub.sum()))
        if piece.shape[0] > 8 and i % 2:  # one deletion and one insertion
            cut = int(rng.integers(1, piece.shape[0] - 4))
            piece = np.concatenate([piece[:cut], piece[cut + int(rng.integers(1, 4)):]])
            ins = int(rng.integers(1, piece.shape[0]))
            piece = np.concatenate([piece[:ins], rng.integers(0, k, 2).astype(np.uint8), piece[ins:]])
        at = int(rng.integers(0, bg.shape[0] + 1))
        seqs.append(np.concatenate([bg[:at], piece, bg[at:]]))
    off = np.concatenate([[0], np.cumsum([len(s) for s in seqs])]).astype(np.int64)
    return np.concatenate(seqs).astype(np.uint8), off


@pytest.mark.parametrize("ge", [1, 2, 3])
@pytest.mark.parametrize("lanes", [4, 8, 16, 32, 64])
def test_exact_instances_all_segment_lengths(A, oracle, lanes, ge):
    from paper_1909_00899_b200.scoring import ScoringScheme

    rng = np.random.default_rng(0xE8AC7 + 131 * lanes + ge)
    k = 20
    mat = rng.integers(-4, 6, (k, k))
    mat = (mat + mat.T) // 2
    mat[np.arange(k), np.arange(k)] = rng.integers(3, 9, k)
    go = ge + int(rng.integers(0, 9))
    sch = ScoringScheme.from_array(mat, go, ge)
    tried = 0
    for L in range(1, 65):
        m = lanes * L - int(rng.integers(0, lanes))  # ceil(m / lanes) == L
        if m < 1:
            m = 1
        q = rng.integers(0, k, m).astype(np.uint8)
        try:
            prof = A.build_profile_arrays(q, sch, lanes)
        except Exception:  # noqa: BLE001 -- no instance for this (lanes, L)
            continue
        if prof.plan16.seg_len != L or prof.plan16.lanes != lanes:
            continue  # the layout fell back to another stripe count: no instance here
        db, off = _targets(rng, q, k)
        sc, rend, qend = oracle.db_scalar(q, db, off, mat, go, ge)
        tgt = torch.from_numpy(db).cuda()
        start = torch.from_numpy(off[:-1].copy()).cuda()
        length = torch.from_numpy(np.diff(off).astype(np.int32)).cuda()
        out = A.db_align(prof, tgt, start, length, None, "scan")
        assert (out["score"].cpu().numpy() == sc).all(), (lanes, L, ge, "score")
        assert (out["ref_end"].cpu().numpy() == rend).all(), (lanes, L, ge, "ref_end")
        assert (out["query_end"].cpu().numpy() == qend).all(), (lanes, L, ge, "query_end")
        # score-only launch (no coordinate outputs: the gate-free path of short segments)
        n = length.shape[0]
        so = {"score": torch.empty(n, dtype=torch.int32, device="cuda"), "ref_end": None,
              "query_end": None, "flags": torch.empty(n, dtype=torch.uint8, device="cuda")}
        A.db_align(prof, tgt, start, length, None, "scan", out=so, rescue=False)
        assert (so["score"].cpu().numpy() == sc).all(), (lanes, L, ge, "score-only")
        tried += 1
    assert tried >= 8, f"only {tried} segment lengths had an instance at {lanes} lanes"


@pytest.mark.parametrize("ge", [1, 2, 3])
def test_exact_pair_instances_uniform_queries_ragged_targets(A, oracle, ge):
    """Pairs mode through the exact instances (uniform query length per batch, so every
    pair has the same segment length) with targets of very different lengths inside one
    warp: the short ones run on the shared null-residue row while their neighbours
    finish.  Every segment length 1..32 at 8 stripes, scores and end coordinates
    against the scalar oracle, with and without coordinate outputs."""
    from paper_1909_00899_b200.scoring import ScoringScheme

    rng = np.random.default_rng(0xA11CE + ge)
    mat = np.full((4, 4), -3, dtype=np.int64)
    np.fill_diagonal(mat, 2)
    go = ge + 4
    sch = ScoringScheme.from_array(mat, go, ge)
    for L in range(1, 33):
        m = 8 * L - int(rng.integers(0, 8))
        m = max(m, 1)
        n = 96
        tl = rng.integers(1, 3 * m + 40, n)
        tl[::7] = 1
        q_off = (np.arange(n + 1) * m).astype(np.int64)
        r_off = np.concatenate([[0], np.cumsum(tl)]).astype(np.int64)
        fr = rng.integers(0, 4, r_off[-1]).astype(np.uint8)
        fq = rng.integers(0, 4, q_off[-1]).astype(np.uint8)
        for i in range(0, n, 2):  # plant a mutated piece of the target in the query
            t = fr[r_off[i]:r_off[i + 1]]
            k = min(len(t), m)
            if k >= 4:
                piece = t[:k].copy()
                piece[rng.random(k) < 0.05] = rng.integers(0, 4)
                fq[q_off[i] + m - k:q_off[i] + m] = piece
        s, re_, qe = oracle.batch_scalar(fq, q_off, fr, r_off, sub=mat, go=go, ge=ge)
        r = A.pairs_align(fq, q_off, fr, r_off, kernel="scan", scheme=sch)
        assert (r["score"] == s).all(), (L, ge, "score")
        assert (r["ref_end"] == re_).all() and (r["query_end"] == qe).all(), (L, ge, "coords")
        so = A.pairs_align(fq, q_off, fr, r_off, kernel="scan", scheme=sch, coords=False)
        assert (so["score"] == s).all(), (L, ge, "score-only")
