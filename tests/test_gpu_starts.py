"""Device start coordinates (align.align_starts, search.hit_starts) against the
oracle's anchored reverse DP (swo_start_coords), exact."""

from __future__ import annotations

import numpy as np
import pytest

from helpers import mm_matrix

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def A():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_00899_b200 import align

    return align


def test_starts_random_pairs(A, oracle):
    from paper_1909_00899_b200.scoring import ScoringScheme

    rng = np.random.default_rng(0x5747)
    for trial in range(6):
        k = int(rng.integers(2, 21))
        mat = rng.integers(-5, 6, (k, k))
        np.fill_diagonal(mat, np.abs(np.diag(mat)) + 1)
        go = int(rng.integers(1, 12))
        ge = int(rng.integers(1, go + 1))
        sch = ScoringScheme.from_array(mat, go, ge)
        n = 300
        ql = rng.integers(1, 300, n)
        tl = rng.integers(1, 500, n)
        q_off = np.concatenate([[0], np.cumsum(ql)]).astype(np.int64)
        r_off = np.concatenate([[0], np.cumsum(tl)]).astype(np.int64)
        fq = rng.integers(0, k, q_off[-1]).astype(np.uint8)
        fr = rng.integers(0, k, r_off[-1]).astype(np.uint8)
        for t in range(0, n, 2):  # plant homologous stretches in half of the pairs
            a = int(min(ql[t] // 2, tl[t] - 3))
            if a > 0:
                fr[r_off[t] + 3: r_off[t] + 3 + a] = fq[q_off[t]: q_off[t] + a]
        s, re_, qe = oracle.batch_scalar(fq, q_off, fr, r_off, sub=mat, go=go, ge=ge)
        want = oracle.batch_starts(fq, q_off, fr, r_off, mat, go, ge, s, re_, qe)
        for width in (16, 32):
            got = A.align_starts(fq, q_off, fr, r_off, sch, s, re_, qe, width=width)
            assert (got[0] == want[0]).all() and (got[1] == want[1]).all(), (trial, width)


def test_starts_config1_and_long_scores(A, oracle):
    from paper_1909_00899_b200 import workloads as W

    w = W.config1()
    sub = w.scheme.as_array()
    s, re_, qe = oracle.scalar(w.query, w.ref, sub, 5, 2)
    q_off = np.array([0, w.query.size], np.int64)
    r_off = np.array([0, w.ref.size], np.int64)
    got = A.align_starts(w.query, q_off, w.ref, r_off, w.scheme, [s], [re_], [qe])
    assert (int(got[0][0]), int(got[1][0])) == oracle.start_coords(w.query, w.ref, sub, 5, 2, s, re_, qe)
    # a score past the 16-bit range: rescued launch, same rule
    q = np.zeros(3000, np.uint8)
    r = np.concatenate([np.ones(50, np.uint8), q, np.ones(50, np.uint8)])
    from paper_1909_00899_b200.scoring import ScoringScheme
    sch = ScoringScheme.from_array(mm_matrix(20, -3, 4), 3, 1)
    s2, re2, qe2 = oracle.scalar(q, r, mm_matrix(20, -3, 4), 3, 1)
    got = A.align_starts(q, [0, q.size], r, [0, r.size], sch, [s2], [re2], [qe2])
    assert s2 == 60_000 and (int(got[0][0]), int(got[1][0])) == (50, 0)


def test_database_topk_hit_starts(A, oracle):
    from paper_1909_00899_b200 import search, workloads

    w2 = workloads.config2(n_targets=3000)
    packed = search.pack(w2.db, w2.offsets)
    eng = search.DatabaseSearch(w2.scheme, coords="topk", k=20)
    eng.set_query(w2.query)
    eng.upload(packed)
    eng.align()
    top = eng.topk(20)
    rec = search.hit_starts(w2.query, top, w2.db, w2.offsets, w2.scheme)
    sub = w2.scheme.as_array()
    for score, tid, rend, qend, rs, qs in rec:
        t = w2.db[w2.offsets[tid]:w2.offsets[tid + 1]]
        assert (rs, qs) == oracle.start_coords(w2.query, t, sub, w2.scheme.gap_open,
                                               w2.scheme.gap_extend, score, rend, qend)
        assert oracle.scalar(w2.query[qs:qend + 1], t[rs:rend + 1], sub, w2.scheme.gap_open,
                             w2.scheme.gap_extend)[0] == score


def test_runner_starts_columns(A, oracle):
    """--starts: TSV gains ref_start/query_start equal to the oracle's."""
    import io

    from paper_1909_00899_b200 import runner

    buf = io.StringIO()
    cfg = runner.RunConfig(random_count=40, seed=9, len_max=120, match=2, mismatch=-3,
                           gap_open=5, gap_extend=2, starts=True)
    assert runner.run(cfg, out=buf) == 0
    lines = [x for x in buf.getvalue().splitlines() if not x.startswith("#")]
    assert lines[0].endswith("ref_end\tquery_end\tref_start\tquery_start")
    alpha, sch = runner._build_scheme(cfg)
    ps = runner.load_pairs(cfg, alpha)
    sub = sch.as_array()
    for i, row in enumerate(lines[1:]):
        f = row.split("\t")
        q = ps.fq[ps.q_off[i]:ps.q_off[i + 1]]
        t = ps.fr[ps.r_off[i]:ps.r_off[i + 1]]
        score, rend, qend = oracle.scalar(q, t, sub, 5, 2)
        assert (int(f[4]), int(f[9]), int(f[10])) == (score, rend, qend)
        assert (int(f[11]), int(f[12])) == oracle.start_coords(q, t, sub, 5, 2, score, rend, qend)
