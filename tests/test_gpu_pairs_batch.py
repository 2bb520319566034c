"""PairsBatch (config 3's device batch): resident and streamed-from-host forms
against the oracle (batch_align / batch_oracle_scores, src/_compiled.py:491-529)."""

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


@pytest.mark.parametrize("lanes", [0, 4])
@pytest.mark.parametrize("coords", [False, True])
def test_pairs_batch_resident_and_streamed(A, oracle, coords, lanes):
    """lanes=0: the throughput layout (8 stripes, 19 words); lanes=4: 4 stripes of 38
    words (T = 2, four groups interleaved per 32-word profile block)."""
    from paper_1909_00899_b200 import workloads as W

    w = W.config3(n_pairs=50_000)
    s, re_, qe = oracle.batch_scalar(w.flat_q, w.q_off, w.flat_r, w.r_off,
                                     sub=w.scheme.as_array(), go=6, ge=1)
    b = A.PairsBatch(w.scheme, coords=coords, lanes=lanes)
    b.upload(w.flat_q, w.q_off, w.flat_r, w.r_off)
    o = b.run()
    assert (o["score"][: w.n_pairs].cpu().numpy() == s).all()
    if coords:
        assert (o["ref_end"][: w.n_pairs].cpu().numpy() == re_).all()
        assert (o["query_end"][: w.n_pairs].cpu().numpy() == qe).all()
    host = A.PairsBatch.pin_host(w.flat_q, w.q_off, w.flat_r, w.r_off)
    e = A.PairsBatch(w.scheme, coords=coords, lanes=lanes)
    e.prepare_host(host, n_chunks=7)
    for _ in range(2):  # buffers are reused across calls
        h = e.run_host(host)
        torch.cuda.synchronize()
        assert (h["score"].numpy() == s).all()
        if coords:
            assert (h["ref_end"].numpy() == re_).all() and (h["query_end"].numpy() == qe).all()


def test_pairs_batch_mixed_lengths_and_rescue(A, oracle):
    """Ragged pairs (empty, 1-residue, up to 300) and a scheme whose scores pass the
    16-bit guard (re-run in 32 bits on the device), resident and streamed."""
    from paper_1909_00899_b200.scoring import ScoringScheme

    rng = np.random.default_rng(0x9A1)
    n = 3000
    ql = rng.integers(0, 300, n)
    tl = rng.integers(0, 400, n)
    ql[:5] = [0, 1, 300, 299, 0]
    tl[:5] = [10, 0, 400, 1, 0]
    q_off = np.concatenate([[0], np.cumsum(ql)]).astype(np.int64)
    r_off = np.concatenate([[0], np.cumsum(tl)]).astype(np.int64)
    fq = rng.integers(0, 4, q_off[-1]).astype(np.uint8)
    fr = rng.integers(0, 4, r_off[-1]).astype(np.uint8)
    fr[r_off[10]:r_off[10] + min(tl[10], ql[10])] = fq[q_off[10]:q_off[10] + min(tl[10], ql[10])]
    mat = np.full((4, 4), -3, np.int8)
    np.fill_diagonal(mat, 120)
    sch = ScoringScheme.from_array(mat, 5, 2)
    s, re_, qe = oracle.batch_scalar(fq, q_off, fr, r_off, sub=mat, go=5, ge=2)
    assert s.max() > 32767 - 120  # some pairs need the 32-bit rescue
    b = A.PairsBatch(sch, coords=True)
    b.upload(fq, q_off, fr, r_off)
    o = b.run()
    assert (o["score"][:n].cpu().numpy() == s).all()
    assert (o["ref_end"][:n].cpu().numpy() == re_).all()
    host = A.PairsBatch.pin_host(fq, q_off, fr, r_off)
    e = A.PairsBatch(sch, coords=True)
    e.prepare_host(host, n_chunks=5)
    h = e.run_host(host)
    torch.cuda.synchronize()
    assert (h["score"].numpy() == s).all() and (h["query_end"].numpy() == qe).all()


def test_database_search_four_stripes(A, oracle):
    """The T = 2 exact instances in database mode (four profile copies interleaved per
    32-word block): a 150-residue query at lanes=4, every target against the oracle."""
    from paper_1909_00899_b200 import search, workloads as W

    w = W.config2(n_targets=3000)
    q = w.query[:150].copy()
    packed = search.pack(w.db, w.offsets, pin=False)
    eng = search.DatabaseSearch(w.scheme, coords="all", lanes=4)
    eng.upload(packed)
    eng.set_query(q)
    assert (eng.plan16.lanes, eng.plan16.seg_len) == (4, 38)
    o = eng.align()
    ids = packed.ids.numpy()
    s, re_, qe = oracle.db_scalar(q, w.db, w.offsets, w.scheme.as_array(), 11, 1)
    assert (o["score"][: w.n_targets].cpu().numpy() == s[ids]).all()
    assert (o["ref_end"][: w.n_targets].cpu().numpy() == re_[ids]).all()
    assert (o["query_end"][: w.n_targets].cpu().numpy() == qe[ids]).all()


def test_pairs_batch_2bit_packed_input(A, oracle):
    """Fixed-length DNA batch from 2-bit packed pinned input (formats.pack_2bit, expanded on
    the device by sw_unpack_2bit): same scores and coordinates as the one-byte input and the
    oracle, a quarter of the H2D bytes; ragged batches are refused."""
    import torch as T

    from paper_1909_00899_b200 import workloads as W
    from paper_1909_00899_b200.formats import pack_2bit, unpack_2bit

    w = W.config3(n_pairs=5000)
    sub = w.scheme.as_array()
    s, re_, qe = oracle.batch_scalar(w.flat_q, w.q_off, w.flat_r, w.r_off, sub=sub,
                                     go=w.scheme.gap_open, ge=w.scheme.gap_extend)
    # the unpack kernel alone, odd lengths included
    L = __import__("paper_1909_00899_b200._lib", fromlist=["load"]).load()
    for n in (1, 3, 4, 5, 1023, 150 * 4999):
        codes = np.ascontiguousarray(w.flat_q[:n])
        d_p = T.from_numpy(pack_2bit(codes)).cuda()
        d_c = T.full((n + 8,), 77, dtype=T.uint8, device="cuda")
        assert L.sw_unpack_2bit(d_p.data_ptr(), n, d_c.data_ptr(), T.cuda.current_stream().cuda_stream) == 0
        got = d_c.cpu().numpy()
        assert (got[:n] == codes).all() and (got[n:] == 77).all(), n
        assert (unpack_2bit(pack_2bit(codes), n) == codes).all()
    for coords in (False, True):
        b = A.PairsBatch(w.scheme, coords=coords)
        host = b.pin_host(w.flat_q, w.q_off, w.flat_r, w.r_off, packed2bit=True)
        b.prepare_host(host, n_chunks=7)
        out = b.run_host(host)
        T.cuda.synchronize()
        assert b.h2d_bytes == (len(w.flat_q) + 3) // 4 + (len(w.flat_r) + 3) // 4
        assert (out["score"].numpy() == s).all()
        if coords:
            assert (out["ref_end"].numpy() == re_).all() and (out["query_end"].numpy() == qe).all()
    ragged = W.config3(n_pairs=64)
    q_off = ragged.q_off.copy()
    q_off[-1] -= 3
    with pytest.raises(ValueError):
        bb = A.PairsBatch(w.scheme)
        bb.prepare_host(bb.pin_host(ragged.flat_q[:q_off[-1]], q_off, ragged.flat_r, ragged.r_off,
                                    packed2bit=True), n_chunks=2)

