"""CPU-side checks of the C ABI library and the host layer (no GPU needed)."""

from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols() -> list[str]:
    with open(os.path.join(REPO, "include", "swscan_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|const char\*)\s+(sw_\w+)\(", text, re.M)))


def test_header_declares_the_exported_api():
    from paper_1909_00899_b200 import _lib

    assert set(_declared_symbols()) == set(_lib.EXPORTS)


def test_library_loads_and_exports_every_declared_symbol():
    from paper_1909_00899_b200 import _lib

    _lib.build()
    lib = C.CDLL(_lib.LIB_PATH)
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    L = _lib.load()
    assert L.sw_version() == 1


def test_plan_reproduces_reference_layout():
    from paper_1909_00899_b200 import _lib

    _lib.build()
    for m in (1, 3, 17, 150, 255, 464):
        for p in (2, 4, 8, 16, 32, 64):
            L = (m + p - 1) // p
            if L > 32:
                with pytest.raises(_lib.SwError):
                    _lib.plan_query(m, 4, 16, p)
                continue
            pl = _lib.plan_query(m, 4, 16, p)
            assert (pl.lanes, pl.threads, pl.seg_len) == (p, p // 2, L)
            assert pl.lmax >= L and pl.prof_words == 5 * L * (p // 2)
    auto = _lib.plan_query(464, 20, 16, 0)  # exact long-segment instance: 8 stripes x 58 words
    assert (auto.lanes, auto.threads, auto.seg_len, auto.lmax) == (8, 4, 58, 58)
    auto = _lib.plan_query(150, 4, 16, 0)
    assert (auto.lanes, auto.threads, auto.seg_len) == (8, 4, 19)
    with pytest.raises(_lib.SwError):
        _lib.plan_query(10, 4, 24, 0)
    with pytest.raises(_lib.SwError):
        _lib.plan_query(10, 4, 16, 6)


def test_block_plan_reference_layouts():
    """Host-side geometry of the block / cluster kernel (sw_block_plan): the
    reference layout VectorSpec(p) beyond one warp, CTAs per cluster chosen to fit
    the per-CTA thread and shared-memory limits, lazy-F on one CTA only."""
    from paper_1909_00899_b200 import _lib

    _lib.build()
    scan, lazy = _lib.KERNEL_IDS["scan"], _lib.KERNEL_IDS["lazyf"]
    for m, p, width, want in ((2048, 2048, 16, (2048, 1024, 1, 1)),
                              (2048, 256, 16, (256, 128, 1, 8)),
                              (65536, 16384, 32, (16384, 1024, 16, 4)),
                              (65536, 4096, 32, (4096, 256, 16, 16)),
                              (8192, 16384, 16, (16384, 1024, 8, 1)),
                              (1000, 128, 32, (128, 128, 1, 8))):
        assert _lib.block_plan(m, 4, width, scan, p) == want, (m, p, width)
    # L = ceil(m / p) must be 1..16; p a power of two of at least one warp pair
    assert _lib.block_plan(4096, 4, 16, scan, 128) is None
    assert _lib.block_plan(100, 4, 16, scan, 96) is None
    assert _lib.block_plan(100, 4, 16, scan, 32) is None
    # lazy-F: one CTA (p <= 2,048 16-bit / 1,024 32-bit)
    assert _lib.block_plan(2048, 20, 16, lazy, 2048) == (2048, 1024, 1, 1)
    assert _lib.block_plan(2048, 20, 32, lazy, 2048) is None
    # a 20-letter profile of 4 words x 1,024 threads exceeds one CTA's shared memory
    assert _lib.block_plan(65536, 20, 32, scan, 16384) is None
    # automatic layout: scan prefers <= 4-word segments, lazy-F the fewest stripes
    assert _lib.block_plan(2048, 20, 16, scan, 0) == (512, 256, 1, 4)
    assert _lib.block_plan(2048, 20, 16, lazy, 0) == (128, 64, 1, 16)


def test_counters_closed_form_matches_reference_tallies(oracle):
    """Host reconstruction of the reference's op counters from pass counts."""
    from paper_1909_00899_b200.align import counters_from_passes

    rng = np.random.default_rng(3)
    sub = np.full((4, 4), -2, np.int8)
    np.fill_diagonal(sub, 3)
    for _ in range(30):
        q = rng.integers(0, 4, int(rng.integers(1, 80)))
        r = rng.integers(0, 4, int(rng.integers(1, 80)))
        p = int(rng.choice([2, 4, 8, 16]))
        for kern in ("scan", "lazyf", "lazyf-noexit"):
            _, _, cnt, colp = oracle.align_pair(kern, p, q, r, sub, 4, 1)
            L = (len(q) + p - 1) // p
            c = counters_from_passes(kern, len(r), L, p, colp)
            assert [c.shifts, c.sat_adds, c.sat_subs, c.maxes, c.loads, c.stores,
                    c.correction_passes] == list(cnt)


def test_scoring_mirrors_reference_validation():
    from paper_1909_00899_b200.scoring import Alphabet, ScoringScheme, SymbolOutOfAlphabet

    with pytest.raises(ValueError):
        ScoringScheme(((1, 2), (3,)), 3, 1)
    with pytest.raises(ValueError):
        ScoringScheme(((200,),), 3, 1)
    with pytest.raises(ValueError):
        ScoringScheme(((1,),), 1, 2)
    dna = Alphabet.dna()
    sch = ScoringScheme.match_mismatch(dna, 2, -3, 5, 2)
    assert sch.bias == 3 and sch.max_score == 2
    assert sch.matrix[4] == (-3,) * 5  # wildcard row scores mismatch
    assert list(dna.encode_array("ACGTN")) == [0, 1, 2, 3, 4]
    with pytest.raises(SymbolOutOfAlphabet):
        dna.encode_array("ACGX")


def test_product_path_has_no_cpu_fallback(monkeypatch):
    """Without a CUDA device the product raises instead of computing on the CPU."""
    import torch

    from paper_1909_00899_b200 import _lib, align
    from paper_1909_00899_b200.scoring import Alphabet, ScoringScheme

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    sch = ScoringScheme.match_mismatch(Alphabet("ACGT"), 2, -1, 3, 1)
    with pytest.raises(_lib.NativeUnavailable):
        align.align_pair("scan", 8, [0, 1, 2], [0, 1], sch)


def _header_arity() -> dict[str, int]:
    with open(os.path.join(REPO, "include", "swscan_b200.h")) as fh:
        text = re.sub(r"/\*.*?\*/", "", fh.read(), flags=re.S)
    out = {}
    for m in re.finditer(r"(?:int32_t|int64_t|const char\*)\s+(sw_\w+)\(([^)]*)\);", text):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    return out


def integration_stub() -> str:
    """The ctypes stub of INTEGRATION.md §2, verbatim."""
    with open(os.path.join(REPO, "INTEGRATION.md")) as fh:
        text = fh.read()
    block = text.split("<!-- stub:begin -->", 1)[1].split("<!-- stub:end -->", 1)[0]
    return block.split("```python", 1)[1].rsplit("```", 1)[0]


def test_integration_stub_signatures(monkeypatch):
    """The documented drop-in stub binds every entry point with the header's arity
    (the old stub passed 23 arguments to the 21-parameter sw_db_align)."""
    from paper_1909_00899_b200 import _lib

    _lib.build()
    monkeypatch.setenv("SWSCAN_B200_LIB", _lib.LIB_PATH)
    ns: dict = {}
    exec(compile(integration_stub(), "INTEGRATION.md", "exec"), ns)
    arity = _header_arity()
    assert arity["sw_db_align"] == 21
    for name in ("sw_plan_query", "sw_profile_build", "sw_db_align"):
        assert len(getattr(ns["_L"], name).argtypes) == arity[name], name
    # and the package's own binding agrees with the header everywhere
    L = _lib.load()
    for name in _lib.EXPORTS:
        assert len(getattr(L._lib, name).argtypes) == arity[name], name
