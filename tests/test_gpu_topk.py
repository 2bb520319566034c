"""The library's device top-k (sw_topk) against torch.topk on the same keys.

Order: score descending, then target id ascending (BASELINE.json config 2's
top-100 merge).  Cases: random scores with many ties, scores beyond the
histogram's 4,095 bins, fewer elements than k, and mass ties (every score equal,
which overflows the candidate list and takes the exact radix-select path).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _want(score, ids, re_, qe, k):
    k = min(k, score.shape[0])
    key = (score.to(torch.int64) << 32) | (0xFFFFFFFF - ids.to(torch.int64))
    _, idx = torch.topk(key, k, sorted=True)
    return torch.stack([score[idx].to(torch.int64), ids[idx], re_[idx].to(torch.int64),
                        qe[idx].to(torch.int64)], dim=1)


@pytest.mark.parametrize("n,k,hi", [(1_000_000, 100, 90), (1_000_000, 100, 70000), (50, 100, 20),
                                    (5000, 1024, 8), (1, 1, 5), (300_000, 100, 1),
                                    (20_000, 37, 40000)])
def test_topk_matches_torch(n, k, hi):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_00899_b200 import search

    g = torch.Generator(device="cpu").manual_seed(n * 31 + k)
    score = torch.randint(0, hi, (n,), generator=g, dtype=torch.int32).cuda()
    ids = torch.randperm(n, generator=g).to(torch.int64).cuda() + 7
    re_ = torch.randint(-2, 5000, (n,), generator=g, dtype=torch.int32).cuda()
    qe = torch.randint(-2, 464, (n,), generator=g, dtype=torch.int32).cuda()
    got = search.topk_records(score, ids, re_, qe, k)
    want = _want(score, ids, re_, qe, k)
    assert got.shape == want.shape
    assert torch.equal(got, want)
    # repeated calls reuse the scratch and stay exact
    got2 = search.topk_records(score, ids, re_, qe, k)
    assert torch.equal(got2, want)


def test_topk_planted_best_and_all_equal():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1909_00899_b200 import search

    n = 400_000
    score = torch.full((n,), 17, dtype=torch.int32).cuda()  # mass ties: radix-select path
    ids = torch.arange(n, dtype=torch.int64).cuda()
    z = torch.zeros(n, dtype=torch.int32).cuda()
    got = search.topk_records(score, ids, z, z, 100)
    assert torch.equal(got[:, 1].cpu(), torch.arange(100))
    assert (got[:, 0] == 17).all()
    score[123456] = 40000
    score[7] = 18
    got = search.topk_records(score, ids, z, z, 100)
    assert got[0].tolist() == [40000, 123456, 0, 0] and got[1].tolist() == [18, 7, 0, 0]
    assert torch.equal(got[2:, 1].cpu(), torch.tensor([i for i in range(99) if i != 7][:98]))
