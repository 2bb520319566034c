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
