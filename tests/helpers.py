"""Test helpers shared by the CPU and GPU suites."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name: str):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".json"):
        with open(path) as fh:
            return json.load(fh)
    return np.load(path)


def sha(*arrays) -> str:
    """Same digest as tests/golden/make_golden.py:sha."""
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def acceptance_sweep_inputs(n=10_000):
    """Regenerates the reference acceptance sweep (tests/test_acceptance.py:47-62)."""
    rng = np.random.default_rng(0xACCE97)
    len_q = rng.integers(1, 257, n)
    len_t = rng.integers(1, 257, n)
    match = rng.integers(1, 5, n)
    mismatch = -rng.integers(1, 5, n)
    gap_open = rng.integers(1, 9, n)
    gap_extend = np.array([int(rng.integers(1, g + 1)) for g in gap_open], dtype=np.int64)
    q_off = np.zeros(n + 1, dtype=np.int64)
    q_off[1:] = np.cumsum(len_q)
    t_off = np.zeros(n + 1, dtype=np.int64)
    t_off[1:] = np.cumsum(len_t)
    flat_q = rng.integers(0, 4, q_off[-1]).astype(np.int16)
    flat_t = rng.integers(0, 4, t_off[-1]).astype(np.int16)
    return flat_q, q_off, flat_t, t_off, match, mismatch, gap_open, gap_extend


def mm_matrix(match: int, mismatch: int, k: int = 4) -> np.ndarray:
    """4x4 match/mismatch matrix as batch_align's _fill_sub4 (src/_compiled.py:483-488)."""
    m = np.full((k, k), mismatch, dtype=np.int8)
    np.fill_diagonal(m, match)
    return m


def result_digest(score, ref_end, query_end, blocks: int = 256) -> dict:
    """Digest of full-size results (tests/golden/make_fullsize.py): sha256 over the
    int32 (score, ref_end, query_end) arrays plus per-block digests (16 hex chars
    each, contiguous blocks of items) so a mismatch is localised."""
    s = np.ascontiguousarray(score, dtype=np.int32)
    r = np.ascontiguousarray(ref_end, dtype=np.int32)
    q = np.ascontiguousarray(query_end, dtype=np.int32)
    n = s.shape[0]
    bounds = [n * b // blocks for b in range(blocks + 1)]
    bd = [sha(s[a:b], r[a:b], q[a:b])[:16] for a, b in zip(bounds[:-1], bounds[1:])]
    return {"n": int(n), "digest": sha(s, r, q), "blocks": blocks, "block_digests": bd,
            "score_sum": int(s.astype(np.int64).sum()), "score_max": int(s.max()) if n else 0}


def digest_mismatch(got: dict, want: dict) -> str:
    """Human-readable difference between two result_digest dicts ('' when equal)."""
    if got["digest"] == want["digest"]:
        return ""
    bad = [i for i, (a, b) in enumerate(zip(got["block_digests"], want["block_digests"])) if a != b]
    return (f"digest differs in {len(bad)} of {want['blocks']} blocks (first {bad[:8]}); "
            f"score sum {got['score_sum']} vs {want['score_sum']}, max {got['score_max']} vs "
            f"{want['score_max']}")
