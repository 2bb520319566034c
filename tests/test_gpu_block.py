"""Device parity of the block / cluster kernel (sw_align_block): the reference layout
VectorSpec(p) for p beyond one warp, with the F scan resolved warp -> block ->
cluster (distributed shared memory), and the block-wide lazy-F.  Exact equality
against the oracle (scores, end coordinates, per-column lazy-F passes)."""

from __future__ import annotations

import numpy as np
import pytest

from helpers import golden, mm_matrix

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def A():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_00899_b200 import align

    return align


def mm(match, mismatch, go, ge, k=4):
    from paper_1909_00899_b200.scoring import ScoringScheme

    return ScoringScheme.from_array(mm_matrix(match, mismatch, k), go, ge)


def _triple(o):
    return (o["score"], o["ref_end"], o["query_end"])


@pytest.mark.parametrize("width", [16, 32])
def test_block_scan_random_layouts(A, oracle, width):
    """Random schemes, ragged query lengths (pads in the last lanes), every block
    and cluster shape from one warp pair up to a 16-CTA cluster."""
    from paper_1909_00899_b200.scoring import ScoringScheme

    rng = np.random.default_rng(0xB10C + width)
    lpw = 2 if width == 16 else 1
    cases = [64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384]
    for trial, p in enumerate(cases * 2):
        if p < 32 * lpw:
            continue
        k = int(rng.integers(2, 21))
        mat = rng.integers(-5, 6, (k, k))
        go = int(rng.integers(1, 12))
        ge = int(rng.integers(1, go + 1))
        sch = ScoringScheme.from_array(mat, go, ge)
        # L = ceil(m / p) in 1..4 (cluster shapes need L <= 4 at 1,024 threads per CTA)
        m = int(rng.integers(max(1, p // 2), 4 * p + 1))
        if (m + p - 1) // p > 16:
            m = 16 * p
        n = int(rng.integers(1, 1500))
        q = rng.integers(0, k, m).astype(np.uint8)
        r = rng.integers(0, k, n).astype(np.uint8)
        if trial % 2:  # a homologous block: long diagonal runs across many lanes
            blk = q[: min(m, n)]
            r[: blk.shape[0]] = blk
        geo = A._lib.block_plan(m, k, width, 2, p)
        if geo is None:
            continue
        want = oracle.scalar(q, r, mat, go, ge)
        got = A.align_block(q, r, sch, p, "scan", width)
        assert _triple(got) == want, (trial, p, m, n, geo)
        assert got["lanes"] == p


def test_block_scan_matches_reference_scan_kernel(A, oracle):
    """The reference's own scan kernel (oracle restatement of _align_scan_c) at the
    same p: scores equal, and equal to the exact scalar score."""
    rng = np.random.default_rng(0x5CA1)
    sch = mm(2, -3, 5, 2)
    sub = sch.as_array()
    for p in (128, 256, 1024, 4096):
        m = int(rng.integers(p // 2, 2 * p))
        q = rng.integers(0, 4, m).astype(np.uint8)
        r = rng.integers(0, 4, m + 1000).astype(np.uint8)
        r[500:500 + m] = q
        ref_score = oracle.align_pair("scan", p, q, r, sub, 5, 2)[0]
        got = A.align_pair("scan", p, q, r, sch)
        assert got.score == ref_score == oracle.scalar(q, r, sub, 5, 2)[0]
        assert got.lanes == p and got.seg_len == (m + p - 1) // p


@pytest.mark.parametrize("p", [128, 256, 512, 1024, 2048])
def test_block_lazyf_pass_counts_match_reference(A, oracle, p):
    """Block-wide lazy-F (one vote per pass) in the parity mode reproduces the
    reference's per-column pass counts (src/_compiled.py:189-217) at p stripes,
    on the adversarial 'A' run family of tests/test_acceptance.py:166-218."""
    sch = mm(10, -3, 2, 1)
    sub = sch.as_array()
    q = np.zeros(1024, dtype=np.uint8)
    for kern in ("lazyf", "lazyf-noexit"):
        want = oracle.align_pair(kern, p, q, q, sub, 2, 1)
        r = A.align_pair(kern + "-mirror", p, q, q, sch)
        assert r.score == want[0] == 10240
        assert r.lanes == p
        assert (np.array(r.column_passes) == want[3]).all(), (kern, p)
        assert [r.counters.shifts, r.counters.sat_adds, r.counters.sat_subs, r.counters.maxes,
                r.counters.loads, r.counters.stores, r.counters.correction_passes] == list(want[2])
        fast = A.align_pair(kern, p, q, q, sch)
        assert (fast.score, fast.ref_end, fast.query_end) == (r.score, r.ref_end, r.query_end)


def test_block_lazyf_random_vs_oracle(A, oracle):
    from paper_1909_00899_b200.scoring import ScoringScheme

    rng = np.random.default_rng(0x1A2F)
    for trial in range(8):
        k = int(rng.integers(2, 21))
        mat = rng.integers(-5, 6, (k, k))
        go = int(rng.integers(1, 12))
        ge = int(rng.integers(1, go + 1))
        sch = ScoringScheme.from_array(mat, go, ge)
        p = int(2 ** rng.integers(7, 12))
        m = int(rng.integers(p // 2, 3 * p))
        n = int(rng.integers(1, 800))
        q = rng.integers(0, k, m).astype(np.uint8)
        r = rng.integers(0, k, n).astype(np.uint8)
        sub = mat
        want = oracle.align_pair("lazyf", p, q, r, sub, go, ge)
        got = A.align_pair("lazyf-mirror", p, q, r, sch)
        assert got.score == want[0] == oracle.scalar(q, r, sub, go, ge)[0], (trial, p, m)
        assert (np.array(got.column_passes) == want[3]).all(), (trial, p, m)
        for width in (16, 32):
            if A._lib.block_plan(m, k, width, 0, p) is None:
                continue  # 32-bit lazy-F needs p <= 1,024 (one CTA)
            o = A.align_block(q, r, sch, p, "lazyf", width)
            assert _triple(o) == oracle.scalar(q, r, mat, go, ge), (trial, p, width)


def test_block_config4_scan_and_lazyf_identical(A, oracle):
    """Config 4 (2,048 W vs 100,000, gap open 2 / extend 1) at high stripe counts:
    block scan and block lazy-F give the oracle's score and end coordinates."""
    from paper_1909_00899_b200 import workloads as W

    g = golden("configs.npz")
    w = W.config4()
    want = oracle.scalar(w.query, w.ref, w.scheme.as_array(), 2, 1)
    assert want[0] == int(g["c4_scalar"])
    for p in (256, 512, 2048):
        for width in (16, 32):
            if A._lib.block_plan(w.m, 20, width, 2, p) is None:
                continue
            o = A.align_block(w.query, w.ref, w.scheme, p, "scan", width)
            assert _triple(o) == want, (p, width)
    o = A.align_block(w.query, w.ref, w.scheme, 2048, "lazyf", 16, col_passes=True)
    assert _triple(o) == want
    # per-column passes on a prefix against the reference's lazy-F at p = 2048
    pre = w.ref[:600]
    ref_p = oracle.align_pair("lazyf", 2048, w.query, pre, w.scheme.as_array(), 2, 1)
    r = A.align_pair("lazyf-mirror", 2048, w.query, pre, w.scheme)
    assert r.score == ref_p[0]
    assert (np.array(r.column_passes) == ref_p[3]).all()


def test_block_cluster_config5_slice(A, oracle):
    """Cluster shapes (8 and 16 CTAs, DSMEM boundary ring) on the config-5 slice."""
    from paper_1909_00899_b200 import workloads as W

    g = golden("configs.npz")
    w = W.config5(m=8192, n=131_072, block=7_500)
    want = oracle.scalar(w.query, w.ref, w.scheme.as_array(), 3, 1)
    assert want[0] == int(g["c5slice_scalar"])
    for width, p in ((32, 8192), (32, 4096), (16, 16384), (16, 8192), (32, 2048)):
        o = A.align_block(w.query, w.ref, w.scheme, p, "scan", width)
        assert _triple(o) == want, (width, p, o)
        assert o["lanes"] == p


def test_block_edge_cases(A, oracle):
    sch = mm(2, -3, 5, 2)
    sub = sch.as_array()
    rng = np.random.default_rng(3)
    # one-residue reference, one-residue query at many stripes, all-mismatch pairs
    for m, n in ((1, 1), (1, 500), (700, 1), (129, 2), (4096, 3)):
        q = rng.integers(0, 4, m).astype(np.uint8)
        r = rng.integers(0, 4, n).astype(np.uint8)
        for p in (128, 1024):
            if A._lib.block_plan(m, 4, 16, 2, p) is None:
                continue
            o = A.align_block(q, r, sch, p, "scan", 16)
            assert _triple(o) == oracle.scalar(q, r, sub, 5, 2), (m, n, p)
    q = np.zeros(300, dtype=np.uint8)
    r = np.ones(300, dtype=np.uint8)
    o = A.align_block(q, r, sch, 256, "scan", 16)
    assert _triple(o) == (0, -1, -1)
    # score-only launch
    o = A.align_block(q, q, sch, 256, "scan", 16, coords=False)
    assert o["score"] == 600 and (o["ref_end"], o["query_end"]) == (-1, -1)


def test_block_overflow_rescue(A):
    """16-bit run past the wrap guard is re-run in 32 bits at the same layout."""
    q = np.zeros(2048, dtype=np.uint8)
    o = A.align_block(q, np.zeros(20_000, dtype=np.uint8), mm(20, -3, 3, 1), 1024, "scan", 16)
    assert o["score"] == 40_960 and (o["ref_end"], o["query_end"]) == (2047, 2047)
    assert o["flags"] & A._lib.FLAG_RESCUED and not o["flags"] & A._lib.FLAG_REF_OVERFLOW
