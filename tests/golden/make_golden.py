"""Generate golden fixtures by running the REFERENCE implementation in this container.

The reference (``swscan``, pure Python + numba) lives read-only at
/root/reference and does not exist on the GPU box, so its outputs are frozen
here as small fixtures that the CPU oracle (oracle/) and the CUDA path are both
checked against. Inputs are regenerated from seeds (numpy PCG64, same image on
both sides) and pinned by a sha256 so drift in the generators is detected.

Usage:  python tests/golden/make_golden.py [--full-config5]

The reference is imported from a scratch copy under /tmp (numba's cache=True
would otherwise write into the read-only mount).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src/swscan"
REF_COPY = "/tmp/swscan_ref_copy"

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/swscan_ref_numba_cache")
sys.dont_write_bytecode = True


def _import_reference():
    dst = os.path.join(REF_COPY, "swscan")
    if not os.path.isdir(dst):
        os.makedirs(REF_COPY, exist_ok=True)
        shutil.copytree(REF_SRC, dst)
    sys.path.insert(0, REF_COPY)
    sys.path.insert(0, REPO)
    import swscan  # noqa: F401
    from swscan import _compiled as C

    C.warmup()
    return swscan, C


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def first_argmax(hmat) -> tuple[int, int]:
    """A10: first cell reaching the best in _sw_scalar_c's loop order
    (reference residue i outer, query q inner), 0-based; (-1,-1) for score 0."""
    best, bi, bq = 0, -1, -1
    for i in range(1, len(hmat)):
        row = hmat[i]
        for q in range(1, len(row)):
            if row[q] > best:
                best, bi, bq = row[q], i - 1, q - 1
    return bi, bq


def acceptance_sweep_inputs(n=10_000):
    """Regenerates tests/test_acceptance.py:47-62 (seed 0xACCE97) exactly."""
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


RUNNER_FASTA_Q = ">q1 first\nACGTACGTTGCA\n>q2\nGGGCCCAAATTTACGT\nacgtnn\n"
RUNNER_FASTA_T = ">t1\nTTGCAACGTACG\n\n>t2 second target\nACGTNACGTTTTGGGCCA\n"
RUNNER_MATRIX = "A C G T N\n 5 -4 -4 -4 -2\n-4  5 -4 -4 -2\n-4 -4  5 -4 -2\n-4 -4 -4  5 -2\n-2 -2 -2 -2 -1\n"


def runner_fixtures() -> None:
    """The reference runner's TSV (src/runner.py:162-191) for seeded random pairs with
    every kernel, and for FASTA files + a matrix file; time_ns is masked later."""
    import io
    import tempfile

    from swscan.runner import RunConfig, run

    out = {}
    for kern in ("scalar", "lazyf", "lazyf-noexit", "scan"):
        for lanes in (8, 16):
            buf = io.StringIO()
            rc = run(RunConfig(kernel=kern, lanes=lanes, random_count=150, seed=11, len_max=200,
                               match=3, mismatch=-2, gap_open=4, gap_extend=1), out=buf)
            assert rc == 0
            out[f"random_{kern}_l{lanes}"] = buf.getvalue()
    with tempfile.TemporaryDirectory() as d:
        paths = {}
        for name, text in (("q.fa", RUNNER_FASTA_Q), ("t.fa", RUNNER_FASTA_T),
                           ("m.txt", RUNNER_MATRIX)):
            paths[name] = os.path.join(d, name)
            with open(paths[name], "w") as fh:
                fh.write(text)
        for kern in ("scan", "lazyf"):
            for mode in ("all-vs-all", "zip"):
                buf = io.StringIO()
                rc = run(RunConfig(kernel=kern, lanes=4, matrix_path=paths["m.txt"],
                                   query_path=paths["q.fa"], target_path=paths["t.fa"],
                                   pairs_mode=mode, gap_open=6, gap_extend=2), out=buf)
                assert rc == 0
                out[f"fasta_{kern}_{mode}"] = buf.getvalue()
    out["inputs"] = {"query_fasta": RUNNER_FASTA_Q, "target_fasta": RUNNER_FASTA_T,
                     "matrix": RUNNER_MATRIX}
    with open(os.path.join(HERE, "runner_tsv.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def config3_fixtures(C, cfg: dict) -> None:
    """Config-3-shaped cases (2,000 pairs of the seeded generator) from the
    reference's batch drivers (src/_compiled.py:491-529)."""
    from paper_1909_00899_b200 import workloads as W

    w3 = W.config3(n_pairs=2000)
    cfg["c3_inputs_sha256"] = np.array(sha(w3.flat_q, w3.q_off, w3.flat_r, w3.r_off))
    n3 = w3.n_pairs
    m3 = np.full(n3, 2, np.int64)
    x3 = np.full(n3, -4, np.int64)
    g3 = np.full(n3, 6, np.int64)
    e3 = np.full(n3, 1, np.int64)
    fq3, fr3 = w3.flat_q.astype(np.int16), w3.flat_r.astype(np.int16)
    cfg["c3_scalar"] = C.batch_oracle_scores(fq3, w3.q_off, fr3, w3.r_off, m3, x3, g3, e3)
    for kid, kern in ((0, "lazyf"), (2, "scan")):
        for p in (8, 16):
            sc, ov, _ = C.batch_align(kid, p, fq3, w3.q_off, fr3, w3.r_off, m3, x3, g3, e3)
            cfg[f"c3_{kern}_p{p}"] = sc.astype(np.int64)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--full-config5", action="store_true",
                    help="also score the full 65,536 x 1,048,576 config 5 (minutes)")
    ap.add_argument("--only-runner", action="store_true",
                    help="only regenerate the runner TSV fixtures")
    ap.add_argument("--only-config3", action="store_true",
                    help="only refresh the config-3 keys of configs.npz")
    args = ap.parse_args()
    swscan, C = _import_reference()
    if args.only_config3:
        cfg = dict(np.load(os.path.join(HERE, "configs.npz")))
        config3_fixtures(C, cfg)
        np.savez_compressed(os.path.join(HERE, "configs.npz"), **cfg)
        print("config 3 fixtures refreshed")
        return
    runner_fixtures()
    if args.only_runner:
        return
    from swscan.kernels import weighted_max_scan
    from swscan.oracle import correct_lazyf_full, scan_sequential, sw_scalar
    from swscan.profile import build_profile
    from swscan.scoring import Alphabet, ScoringScheme
    from swscan.vectors import ScoreVector, VectorSpec

    from paper_1909_00899_b200 import workloads as W

    DNA4 = Alphabet("ACGT")
    DNA_N = Alphabet.dna()

    def mm(match=2, mismatch=-1, gap_open=3, gap_extend=1, alphabet=DNA4):
        return ScoringScheme.match_mismatch(alphabet, match, mismatch, gap_open, gap_extend)

    def sv(*v):
        return ScoreVector(tuple(v))

    t0 = time.time()
    manifest = {"generated_by": "tests/golden/make_golden.py", "reference": REF_SRC}

    # ---- A. known-answer tests (inputs from the reference's own tests) ----
    kat = {"scalar": [], "kernels": [], "scan": [], "correction": [], "profile": []}
    for q, r, sch, src in [
        ("AAA", "AA", mm(), "tests/test_oracle.py:61-65"),
        ("ACGT", "AGT", mm(), "tests/test_oracle.py:68-69"),
        ("", "ACGT", mm(), "tests/test_oracle.py:54-58"),
        ("ACGT", "", mm(), "tests/test_oracle.py:54-58"),
        ("ACGT", "TGCA", mm(), "tests/test_oracle.py:80"),
    ]:
        qe, re_ = DNA4.encode(q), DNA4.encode(r)
        score, dp = sw_scalar(qe, re_, sch)
        ri, qi = first_argmax(dp.h)
        kat["scalar"].append({"query": qe, "ref": re_, "matrix": [list(x) for x in sch.matrix],
                              "go": sch.gap_open, "ge": sch.gap_extend, "score": score,
                              "ref_end": ri, "query_end": qi, "source": src})
    n_over = 65535 // 127 + 2
    sch = mm(match=127, mismatch=-1, gap_open=3, gap_extend=1)
    kat["scalar"].append({"query": [0] * n_over, "ref": [0] * n_over,
                          "matrix": [list(x) for x in sch.matrix], "go": 3, "ge": 1,
                          "score": int(C.scalar_score(np.zeros(n_over, np.int16),
                                                      np.zeros(n_over, np.int16), sch)),
                          "ref_end": n_over - 1, "query_end": n_over - 1,
                          "source": "tests/test_oracle.py:128-134"})
    for q, r in [("AAA", "AA"), ("ACGT", "AGT")]:
        for p in (2, 4, 8):
            for kern in ("lazyf", "lazyf-noexit", "scan"):
                res = C.align_pair(kern, p, np.array(DNA4.encode(q), np.int16),
                                   np.array(DNA4.encode(r), np.int16), mm())
                kat["kernels"].append({"query": DNA4.encode(q), "ref": DNA4.encode(r),
                                       "p": p, "kernel": kern, "score": res.score,
                                       "overflow": res.overflow,
                                       "counters": [int(x) for x in (
                                           res.counters.shifts, res.counters.sat_adds,
                                           res.counters.sat_subs, res.counters.maxes,
                                           res.counters.loads, res.counters.stores,
                                           res.counters.correction_passes)],
                                       "column_passes": list(res.column_passes),
                                       "source": "tests/test_kernels.py:154-168"})
    for f, d in [((10, 0, 0, 0), 2), ((5, 9, 1, 7), 3), ((1, 2, 3, 4), 0), ((0, 0, 0, 0), 5),
                 ((65535, 65535, 0, 0), 65545)]:
        spec = VectorSpec(4)
        kat["scan"].append({"f": list(f), "d": d,
                            "weighted": list(weighted_max_scan(sv(*f), d, spec).lanes),
                            "sequential": list(scan_sequential(sv(*f), d, spec).lanes),
                            "source": "tests/test_kernels.py:95-99, tests/test_oracle.py:176-216"})
    out = correct_lazyf_full(sv(10, 0, 0, 0), [sv(0, 0, 0, 0), sv(0, 0, 0, 0)], 1, VectorSpec(4))
    kat["correction"].append({"f": [10, 0, 0, 0], "h": [[0] * 4, [0] * 4], "ge": 1, "p": 4,
                              "out": [list(v.lanes) for v in out],
                              "source": "tests/test_oracle.py:146-149"})
    sch = mm(match=2, mismatch=-1, alphabet=DNA_N)
    prof = build_profile(DNA_N.encode("ACG"), sch, VectorSpec(4))
    kat["profile"].append({"query": DNA_N.encode("ACG"), "matrix": [list(x) for x in sch.matrix],
                           "p": 4, "seg_len": prof.seg_len, "bias": prof.bias,
                           "vectors": [[list(v.lanes) for v in row] for row in prof.vectors],
                           "source": "tests/test_profile.py:21-30"})
    with open(os.path.join(HERE, "kat.json"), "w") as fh:
        json.dump(kat, fh, indent=1)

    # ---- B. first-argmax coordinates from the reference's own H matrices ----
    rng = np.random.default_rng(0xC00D)
    rows = []
    for _ in range(400):
        m = int(rng.integers(1, 33))
        n = int(rng.integers(1, 33))
        k = 4
        q = rng.integers(0, k, m)
        r = rng.integers(0, k, n)
        sch = mm(match=int(rng.integers(1, 5)), mismatch=-int(rng.integers(0, 5)),
                 gap_open=int(rng.integers(1, 7)), gap_extend=1)
        ge = int(rng.integers(1, sch.gap_open + 1))
        sch = ScoringScheme(sch.matrix, sch.gap_open, ge)
        score, dp = sw_scalar(list(q), list(r), sch)
        ri, qi = first_argmax(dp.h)
        rows.append((q, r, sch, score, ri, qi))
    q_off = np.cumsum([0] + [len(x[0]) for x in rows]).astype(np.int64)
    r_off = np.cumsum([0] + [len(x[1]) for x in rows]).astype(np.int64)
    np.savez_compressed(
        os.path.join(HERE, "coords_small.npz"),
        flat_q=np.concatenate([x[0] for x in rows]).astype(np.uint8), q_off=q_off,
        flat_r=np.concatenate([x[1] for x in rows]).astype(np.uint8), r_off=r_off,
        match=np.array([x[2].matrix[0][0] for x in rows], np.int64),
        mismatch=np.array([x[2].matrix[0][1] for x in rows], np.int64),
        go=np.array([x[2].gap_open for x in rows], np.int64),
        ge=np.array([x[2].gap_extend for x in rows], np.int64),
        score=np.array([x[3] for x in rows], np.int64),
        ref_end=np.array([x[4] for x in rows], np.int32),
        query_end=np.array([x[5] for x in rows], np.int32))

    # ---- C. the acceptance sweep (tests/test_acceptance.py:40-76) ----
    fq, qo, ft, to, match, mis, go_a, ge_a = acceptance_sweep_inputs()
    oracle = C.batch_oracle_scores(fq, qo, ft, to, match, mis, go_a, ge_a)
    sweep = {"inputs_sha256": np.array(sha(fq, qo, ft, to, match, mis, go_a, ge_a)),
             "oracle": oracle.astype(np.int64)}
    for kid, kern in enumerate(("lazyf", "lazyf-noexit", "scan")):
        for p in (2, 4, 8, 16):
            sc, ov, cnt = C.batch_align(kid, p, fq, qo, ft, to, match, mis, go_a, ge_a)
            key = f"{kern}_p{p}"
            sweep[f"score_{key}"] = sc.astype(np.int64)
            sweep[f"overflow_{key}"] = ov.astype(np.uint8)
            sweep[f"counters_{key}"] = cnt[:500].astype(np.int64)
    np.savez_compressed(os.path.join(HERE, "acceptance_sweep.npz"), **sweep)

    # ---- D. scan vectors (criterion 3 pattern, seed 0x5CA9) ----
    rng = np.random.default_rng(0x5CA9)
    scan = {}
    for p in (2, 4, 8, 16, 32, 64):
        d = rng.integers(0, 70_000, 256)
        f = rng.integers(0, 65_536, 256 * p).astype(np.uint16).reshape(256, p)
        got = np.stack([C._weighted_max_scan_c(f[i], np.int64(d[i]), np.int64(p))
                        for i in range(256)])
        seq = np.stack([C._scan_sequential_c(f[i], np.int64(d[i]), np.int64(p))
                        for i in range(256)])
        assert (got == seq).all()
        scan[f"f_p{p}"], scan[f"d_p{p}"], scan[f"out_p{p}"] = f, d.astype(np.int64), got
    np.savez_compressed(os.path.join(HERE, "scan_vectors.npz"), **scan)

    # ---- E. adversarial lazy-F family (criterion 4) ----
    sch = mm(match=10, mismatch=-3, gap_open=2, gap_extend=1)
    q = np.zeros(1024, dtype=np.int16)
    adv = {"scalar": np.int64(C.scalar_score(q, q, sch))}
    for p in (8, 16, 32, 64):
        for kern in ("lazyf", "lazyf-noexit", "scan"):
            res = C.align_pair(kern, p, q, q, sch)
            key = f"{kern}_p{p}"
            adv[f"score_{key}"] = np.int64(res.score)
            adv[f"passes_{key}"] = np.array(res.column_passes, dtype=np.int32)
            c = res.counters
            adv[f"counters_{key}"] = np.array([c.shifts, c.sat_adds, c.sat_subs, c.maxes,
                                               c.loads, c.stores, c.correction_passes], np.int64)
    np.savez_compressed(os.path.join(HERE, "adversarial.npz"), **adv)

    # ---- F. configuration-shaped cases from the product's seeded generators ----
    def scheme_of(wl):
        return ScoringScheme(wl.scheme.matrix, wl.scheme.gap_open, wl.scheme.gap_extend)

    cfg = {}
    w1 = W.config1()
    s1 = scheme_of(w1)
    q16, r16 = w1.query.astype(np.int16), w1.ref.astype(np.int16)
    cfg["c1_inputs_sha256"] = np.array(sha(w1.query, w1.ref))
    cfg["c1_scalar"] = np.int64(C.scalar_score(q16, r16, s1))
    for p in (16, 64):
        for kern in ("lazyf", "scan"):
            res = C.align_pair(kern, p, q16, r16, s1)
            cfg[f"c1_{kern}_p{p}_score"] = np.int64(res.score)
            cfg[f"c1_{kern}_p{p}_overflow"] = np.uint8(res.overflow)
            cfg[f"c1_{kern}_p{p}_passes"] = np.array(res.column_passes, np.int32)

    w2 = W.config2(n_targets=300)
    s2 = scheme_of(w2)
    cfg["c2_inputs_sha256"] = np.array(sha(w2.query, w2.db, w2.offsets))
    q16 = w2.query.astype(np.int16)
    prof16, bias16 = C.build_profile_arrays(q16, s2, 16)
    sc2, scan2, lz2 = [], [], []
    for t in range(w2.n_targets):
        r = w2.db[w2.offsets[t]:w2.offsets[t + 1]].astype(np.int16)
        sc2.append(C.scalar_score(q16, r, s2))
        scan2.append(C.align_prebuilt("scan", prof16, bias16, r, s2).score)
        lz2.append(C.align_prebuilt("lazyf", prof16, bias16, r, s2).score)
    cfg["c2_scalar"] = np.array(sc2, np.int64)
    cfg["c2_scan_p16"] = np.array(scan2, np.int64)
    cfg["c2_lazyf_p16"] = np.array(lz2, np.int64)

    config3_fixtures(C, cfg)
    w4 = W.config4()
    s4 = scheme_of(w4)
    q16, r16 = w4.query.astype(np.int16), w4.ref.astype(np.int16)
    cfg["c4_inputs_sha256"] = np.array(sha(w4.query, w4.ref))
    cfg["c4_scalar"] = np.int64(C.scalar_score(q16, r16, s4))
    for kern in ("lazyf", "scan"):
        res = C.align_pair(kern, 64, q16, r16, s4)
        cfg[f"c4_{kern}_p64_score"] = np.int64(res.score)
        cfg[f"c4_{kern}_p64_passes"] = np.array(res.column_passes, np.int16)

    w5 = W.config5(m=8192, n=131_072, block=7_500)
    s5 = scheme_of(w5)
    q16, r16 = w5.query.astype(np.int16), w5.ref.astype(np.int16)
    cfg["c5slice_inputs_sha256"] = np.array(sha(w5.query, w5.ref))
    cfg["c5slice_scalar"] = np.int64(C.scalar_score(q16, r16, s5))
    cfg["c5slice_scan_p64"] = np.int64(C.align_pair("scan", 64, q16, r16, s5).score)
    if args.full_config5:
        w5 = W.config5()
        q16, r16 = w5.query.astype(np.int16), w5.ref.astype(np.int16)
        cfg["c5_inputs_sha256"] = np.array(sha(w5.query, w5.ref))
        res = C.align_pair("scan", 64, q16, r16, s5)
        cfg["c5_scan_p64_score"] = np.int64(res.score)
        cfg["c5_scan_p64_overflow"] = np.uint8(res.overflow)
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **cfg)

    manifest["seconds"] = round(time.time() - t0, 1)
    manifest["files"] = sorted(f for f in os.listdir(HERE) if f.endswith((".npz", ".json"))
                               and f != "manifest.json")
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print(json.dumps(manifest))


if __name__ == "__main__":
    main()
