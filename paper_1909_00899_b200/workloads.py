"""Seeded synthetic inputs for the five BASELINE.json configurations.

None of the configurations uses a public dataset: each is generated here from
a fixed, documented seed with numpy PCG64 (the generator family the reference
uses, src/runner.py:46-69). Choices the configuration text leaves open are
fixed once here (SURVEY §8(d) "Under-specified config details") and documented
in DESIGN.md:

* substitutions are Bernoulli per position and always pick a *different* base;
* indels are Bernoulli per position, insertion or deletion with equal
  probability, length uniform in 1..3;
* BLOSUM62 and the Robinson-Robinson background frequencies are not in this
  container, so configs 2 and 4 use a seeded synthetic stand-in matrix
  (symmetric 20x20, positive diagonal, W/W the largest entry) and a seeded
  Dirichlet composition, labelled ``"synthetic-stand-in"`` in every result.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .scoring import Alphabet, ScoringScheme

DNA4 = Alphabet("ACGT")  # batch_align's 4x4 DNA alphabet (src/_compiled.py:483-488)
AMINO20 = Alphabet("ARNDCQEGHILKMFPSTWYV")
W_CODE = AMINO20.index_of("W")

SEEDS = {1: 0x5EED01, 2: 0x5EED02, 3: 0x5EED03, 4: 0x5EED04, 5: 0x5EED05}
STANDIN_MATRIX_SEED = 0xB10562
STANDIN_COMPOSITION_SEED = 0xC0A1


def standin_protein_matrix() -> np.ndarray:
    """Seeded symmetric 20x20 stand-in for BLOSUM62 (labelled synthetic).

    Off-diagonal entries in -4..3 skewed negative so the expected score of a
    random residue pair is about -1 (BLOSUM62's is about -0.95 at background
    frequencies); diagonal 4..9 with W/W = 11 the largest entry."""
    rng = np.random.default_rng(STANDIN_MATRIX_SEED)
    vals = np.arange(-4, 4)
    probs = np.array([0.08, 0.22, 0.22, 0.20, 0.13, 0.08, 0.05, 0.02])
    off = rng.choice(vals, size=(20, 20), p=probs)
    upper = np.triu(off, 1)
    mat = upper + upper.T
    mat[np.diag_indices(20)] = rng.integers(4, 10, 20)
    mat[W_CODE, W_CODE] = 11
    return mat.astype(np.int8)


def standin_composition() -> np.ndarray:
    """Seeded Dirichlet background composition over AMINO20 (labelled synthetic)."""
    rng = np.random.default_rng(STANDIN_COMPOSITION_SEED)
    return rng.dirichlet(np.full(20, 8.0))


def _draw_codes(rng: np.random.Generator, n: int, probs: np.ndarray | None, k: int) -> np.ndarray:
    """n i.i.d. codes in [0, k): uniform, or by inverse CDF over a 2^16 table."""
    if probs is None:
        return rng.integers(0, k, n, dtype=np.uint8)
    cdf = np.cumsum(probs)
    cdf[-1] = 1.0
    table = np.searchsorted(cdf, (np.arange(65536) + 0.5) / 65536.0).astype(np.uint8)
    out = np.empty(n, dtype=np.uint8)
    step = 1 << 26
    for s in range(0, n, step):
        e = min(n, s + step)
        out[s:e] = table[rng.integers(0, 65536, e - s, dtype=np.uint16)]
    return out


def mutate(seq: np.ndarray, rng: np.random.Generator, sub_rate: float, indel_rate: float,
           k: int) -> np.ndarray:
    """Copy ``seq`` with Bernoulli substitutions (always to a different code)
    and Bernoulli indels (ins/del 50:50, length 1..3)."""
    out = seq.copy()
    subs = rng.random(out.shape[0]) < sub_rate
    out[subs] = (out[subs] + rng.integers(1, k, int(subs.sum()))) % k
    if indel_rate <= 0:
        return out.astype(np.uint8)
    ev = np.flatnonzero(rng.random(out.shape[0]) < indel_rate)
    pieces, prev = [], 0
    for pos in ev:
        pos = int(pos)
        if pos < prev:
            continue
        length = int(rng.integers(1, 4))
        if rng.random() < 0.5:  # insertion before pos
            pieces.append(out[prev:pos])
            pieces.append(rng.integers(0, k, length).astype(out.dtype))
            prev = pos
        else:  # deletion of [pos, pos+length)
            pieces.append(out[prev:pos])
            prev = min(out.shape[0], pos + length)
    pieces.append(out[prev:])
    return np.concatenate(pieces).astype(np.uint8)


@dataclass
class PairWorkload:
    """One query against one reference (configs 1, 4, 5)."""

    name: str
    query: np.ndarray
    ref: np.ndarray
    scheme: ScoringScheme
    alphabet: Alphabet
    width: int
    seed: int
    notes: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.query.shape[0])

    @property
    def cells(self) -> int:
        return int(self.query.shape[0]) * int(self.ref.shape[0])


@dataclass
class DbWorkload:
    """One query against a CSR database of targets (config 2)."""

    name: str
    query: np.ndarray
    db: np.ndarray  # uint8 residues, concatenated
    offsets: np.ndarray  # int64[n+1]
    scheme: ScoringScheme
    alphabet: Alphabet
    seed: int
    notes: dict = field(default_factory=dict)

    @property
    def n_targets(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def cells(self) -> int:
        return int(self.query.shape[0]) * int(self.offsets[-1])


@dataclass
class BatchWorkload:
    """Independent (query_k, target_k) pairs in CSR form (config 3)."""

    name: str
    flat_q: np.ndarray
    q_off: np.ndarray
    flat_r: np.ndarray
    r_off: np.ndarray
    scheme: ScoringScheme
    alphabet: Alphabet
    seed: int
    notes: dict = field(default_factory=dict)

    @property
    def n_pairs(self) -> int:
        return int(self.q_off.shape[0] - 1)

    @property
    def cells(self) -> int:
        return int(np.dot(np.diff(self.q_off), np.diff(self.r_off)))


def config1(seed: int = SEEDS[1]) -> PairWorkload:
    """Single pair DNA 150 x 10,000, query planted with 5% substitutions."""
    rng = np.random.default_rng(seed)
    query = rng.integers(0, 4, 150, dtype=np.uint8)
    ref = rng.integers(0, 4, 10_000, dtype=np.uint8)
    off = int(rng.integers(0, ref.shape[0] - 150 + 1))
    ref[off:off + 150] = mutate(query, rng, 0.05, 0.0, 4)
    scheme = ScoringScheme.match_mismatch(DNA4, 2, -3, 5, 2)
    return PairWorkload("config1-single-pair-dna", query, ref, scheme, DNA4, 16, seed,
                        {"plant_offset": off})


def config2(n_targets: int = 1_000_000, seed: int = SEEDS[2]) -> DbWorkload:
    """Protein DB: query 464 vs lognormal(median 300, sigma 0.6) targets clipped 30..5000."""
    rng = np.random.default_rng(seed)
    comp = standin_composition()
    query = _draw_codes(rng, 464, comp, 20)
    lens = np.clip(np.rint(rng.lognormal(np.log(300.0), 0.6, n_targets)), 30, 5000).astype(np.int64)
    offsets = np.zeros(n_targets + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    db = _draw_codes(rng, int(offsets[-1]), comp, 20)
    scheme = ScoringScheme.from_array(standin_protein_matrix(), 11, 1)
    return DbWorkload("config2-protein-db", query, db, offsets, scheme, AMINO20, seed,
                      {"matrix": "synthetic-stand-in (BLOSUM62 not in container)",
                       "composition": "synthetic-stand-in (Robinson-Robinson not in container)"})


C3_CHUNK = 1 << 16  # config 3 pairs per independently seeded generator block


def config3(n_pairs: int = 1 << 24, seed: int = SEEDS[3], start: int = 0,
            stop: int | None = None, threads: int = 0) -> BatchWorkload:
    """Short reads: 150 nt read vs 300 nt window, 1% subs, 0.1% indels (1..3).

    Pairs are generated in blocks of C3_CHUNK, block b from its own generator
    ``default_rng((seed, b))``, so any pair range [start, stop) -- a rank's shard
    -- is generated without the pairs before it, and a smaller n_pairs is a prefix
    of the full batch. Returns the pairs [start, stop) (default: all n_pairs)."""
    import os

    threads = threads or min(8, os.cpu_count() or 1)
    stop = n_pairs if stop is None else min(stop, n_pairs)
    start = max(0, min(start, stop))
    W, R = 300, 150
    n_out = stop - start
    flat_r = np.empty(n_out * W, dtype=np.uint8)
    flat_q = np.empty(n_out * R, dtype=np.uint8)
    def make_block(blk: int) -> None:
        rng = np.random.default_rng((seed, blk))
        b0 = blk * C3_CHUNK
        n = min(C3_CHUNK, n_pairs - b0)
        win = rng.integers(0, 4, (n, W), dtype=np.uint8)
        off = rng.integers(0, W - R - 16 + 1, n)
        # indel events: per read position, Bernoulli(0.001); type and length
        ev = rng.random((n, R)) < 0.001
        is_ins = rng.random((n, R)) < 0.5
        ln = rng.integers(1, 4, (n, R))
        ins_flag = np.zeros((n, R), dtype=bool)
        ins_ev = ev & is_ins
        for d in range(3):
            sh = np.zeros((n, R), dtype=bool)
            sh[:, d:] = ins_ev[:, :R - d] & (ln[:, :R - d] > d)
            ins_flag |= sh
        dels = np.where(ev & ~is_ins, ln, 0)
        consumed = np.cumsum(~ins_flag, axis=1) - (~ins_flag)
        src = off[:, None] + consumed + np.cumsum(dels, axis=1)
        oob = src >= W
        src = np.minimum(src, W - 1)
        read = np.take_along_axis(win, src, axis=1)
        rnd = rng.integers(0, 4, (n, R), dtype=np.uint8)
        use_rnd = ins_flag | oob
        read[use_rnd] = rnd[use_rnd]
        subs = rng.random((n, R)) < 0.01
        read[subs] = (read[subs] + rng.integers(1, 4, int(subs.sum()))) % 4
        a, b = max(start, b0), min(stop, b0 + n)  # the part of this block in [start, stop)
        flat_r[(a - start) * W:(b - start) * W] = win[a - b0:b - b0].reshape(-1)
        flat_q[(a - start) * R:(b - start) * R] = read[a - b0:b - b0].reshape(-1)

    blocks = range(start // C3_CHUNK, -(-stop // C3_CHUNK))
    if threads > 1 and len(blocks) > 1:  # blocks are independent; numpy releases the GIL
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(min(threads, len(blocks))) as ex:
            list(ex.map(make_block, blocks))
    else:
        for blk in blocks:
            make_block(blk)
    q_off = np.arange(n_out + 1, dtype=np.int64) * R
    r_off = np.arange(n_out + 1, dtype=np.int64) * W
    scheme = ScoringScheme.match_mismatch(DNA4, 2, -4, 6, 1)
    return BatchWorkload("config3-short-reads", flat_q, q_off, flat_r, r_off, scheme, DNA4, seed,
                         {"read_len": R, "window": W, "pairs": [start, stop],
                          "n_pairs_total": n_pairs})


def config4(n_ref: int = 100_000, m: int = 2048, seed: int = SEEDS[4]) -> PairWorkload:
    """Adversarial F: 2048 'W' vs 100,000 uniform amino acids with 10% in W runs."""
    rng = np.random.default_rng(seed)
    query = np.full(m, W_CODE, dtype=np.uint8)
    ref = rng.integers(0, 20, n_ref, dtype=np.uint8)
    in_run = np.zeros(n_ref, dtype=bool)
    target = int(np.ceil(0.10 * n_ref))
    while int(in_run.sum()) < target:
        start = int(rng.integers(0, n_ref))
        length = int(rng.geometric(1.0 / 40.0))
        in_run[start:start + length] = True
    ref[in_run] = W_CODE
    scheme = ScoringScheme.from_array(standin_protein_matrix(), 2, 1)
    return PairWorkload("config4-adversarial-f", query, ref, scheme, AMINO20, 32, seed,
                        {"matrix": "synthetic-stand-in (BLOSUM62 not in container)",
                         "w_run_fraction": float(in_run.mean())})


def config5(m: int = 65_536, n: int = 1_048_576, block: int = 60_000,
            seed: int = SEEDS[5]) -> PairWorkload:
    """Long pair 65,536 x 1,048,576 with a 60,000 nt homologous block (10% subs, 1% indels)."""
    rng = np.random.default_rng(seed)
    query = rng.integers(0, 4, m, dtype=np.uint8)
    ref = rng.integers(0, 4, n, dtype=np.uint8)
    block = min(block, m)
    qo = int(rng.integers(0, m - block + 1))
    hom = mutate(query[qo:qo + block], rng, 0.10, 0.01, 4)
    hom = hom[: min(hom.shape[0], n)]
    ro = int(rng.integers(0, n - hom.shape[0] + 1))
    ref[ro:ro + hom.shape[0]] = hom
    scheme = ScoringScheme.match_mismatch(DNA4, 1, -1, 3, 1)
    return PairWorkload("config5-long-pair", query, ref, scheme, DNA4, 32, seed,
                        {"query_block_offset": qo, "ref_block_offset": ro,
                         "block_len": int(hom.shape[0])})
