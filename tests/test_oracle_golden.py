"""Pin the CPU oracle (oracle/sw_oracle.c) against the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference swscan
package (tests/golden/make_golden.py). Every comparison is exact (tolerance 0):
scores, overflow flags, the seven op counters, per-column pass counts, scan
vectors and first-max end coordinates.
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import acceptance_sweep_inputs, golden, mm_matrix, sha

from paper_1909_00899_b200 import workloads as W


def test_kat_scalar_scores_and_coordinates(oracle):
    for case in golden("kat.json")["scalar"]:
        sub = np.array(case["matrix"], dtype=np.int8)
        score, ri, qi = oracle.scalar(case["query"], case["ref"], sub, case["go"], case["ge"])
        assert score == case["score"], case["source"]
        assert (ri, qi) == (case["ref_end"], case["query_end"]), case["source"]


def test_kat_striped_kernels_scores_counters_passes(oracle):
    sub = mm_matrix(2, -1)
    for case in golden("kat.json")["kernels"]:
        score, ov, cnt, colp = oracle.align_pair(case["kernel"], case["p"], case["query"],
                                                 case["ref"], sub, 3, 1)
        assert score == case["score"]
        assert ov == case["overflow"]
        assert list(cnt) == case["counters"]
        assert list(colp) == case["column_passes"]


def test_kat_scans_and_profile(oracle):
    kat = golden("kat.json")
    for case in kat["scan"]:
        assert list(oracle.weighted_max_scan(case["f"], case["d"])) == case["weighted"]
        assert list(oracle.scan_sequential(case["f"], case["d"])) == case["sequential"]
    for case in kat["profile"]:
        prof, bias = oracle.build_profile(case["query"], np.array(case["matrix"]), case["p"])
        assert bias == case["bias"]
        assert prof.shape[1] == case["seg_len"]
        assert prof.tolist() == case["vectors"]


def test_first_max_coordinates_against_reference_dp_matrices(oracle):
    g = golden("coords_small.npz")
    score, rend, qend = oracle.batch_scalar(g["flat_q"], g["q_off"], g["flat_r"], g["r_off"],
                                            match_a=g["match"], mis_a=g["mismatch"],
                                            go_a=g["go"], ge_a=g["ge"])
    assert (score == g["score"]).all()
    assert (rend == g["ref_end"]).all()
    assert (qend == g["query_end"]).all()


@pytest.fixture(scope="module")
def sweep():
    g = golden("acceptance_sweep.npz")
    inputs = acceptance_sweep_inputs()
    assert sha(*inputs) == str(g["inputs_sha256"]), "acceptance-sweep regeneration drifted"
    return g, inputs


def test_acceptance_sweep_scalar_oracle(oracle, sweep):
    g, (fq, qo, ft, to, match, mis, go_a, ge_a) = sweep
    score, _, _ = oracle.batch_scalar(fq, qo, ft, to, match_a=match, mis_a=mis, go_a=go_a,
                                      ge_a=ge_a)
    assert (score == g["oracle"]).all()


@pytest.mark.parametrize("kernel", ["lazyf", "lazyf-noexit", "scan"])
@pytest.mark.parametrize("p", [2, 4, 8, 16])
def test_acceptance_sweep_striped_kernels(oracle, sweep, kernel, p):
    g, (fq, qo, ft, to, match, mis, go_a, ge_a) = sweep
    score, over, cnt = oracle.batch_striped(kernel, p, fq, qo, ft, to, match_a=match,
                                            mis_a=mis, go_a=go_a, ge_a=ge_a)
    key = f"{kernel}_p{p}"
    assert (score == g[f"score_{key}"]).all()
    assert (over == g[f"overflow_{key}"]).all()
    assert (cnt[:500] == g[f"counters_{key}"]).all()
    assert (score == g["oracle"]).all()


def test_scan_vectors(oracle):
    g = golden("scan_vectors.npz")
    for p in (2, 4, 8, 16, 32, 64):
        f, d, want = g[f"f_p{p}"], g[f"d_p{p}"], g[f"out_p{p}"]
        for i in range(f.shape[0]):
            assert (oracle.weighted_max_scan(f[i], int(d[i])) == want[i]).all()
            assert (oracle.scan_sequential(f[i], int(d[i])) == want[i]).all()


def test_adversarial_lazyf_family(oracle):
    g = golden("adversarial.npz")
    sub = mm_matrix(10, -3)
    q = np.zeros(1024, dtype=np.uint8)
    assert oracle.scalar(q, q, sub, 2, 1)[0] == int(g["scalar"])
    for p in (8, 16, 32, 64):
        for kern in ("lazyf", "lazyf-noexit", "scan"):
            score, _, cnt, colp = oracle.align_pair(kern, p, q, q, sub, 2, 1)
            key = f"{kern}_p{p}"
            assert score == int(g[f"score_{key}"])
            assert (cnt == g[f"counters_{key}"]).all()
            assert (colp == g[f"passes_{key}"]).all()


def test_config_shaped_cases(oracle):
    g = golden("configs.npz")
    w1 = W.config1()
    assert sha(w1.query, w1.ref) == str(g["c1_inputs_sha256"])
    sub = w1.scheme.as_array()
    go, ge = w1.scheme.gap_open, w1.scheme.gap_extend
    assert oracle.scalar(w1.query, w1.ref, sub, go, ge)[0] == int(g["c1_scalar"])
    for p in (16, 64):
        for kern in ("lazyf", "scan"):
            score, ov, _, colp = oracle.align_pair(kern, p, w1.query, w1.ref, sub, go, ge)
            assert score == int(g[f"c1_{kern}_p{p}_score"])
            assert (colp == g[f"c1_{kern}_p{p}_passes"]).all()

    w2 = W.config2(n_targets=300)
    assert sha(w2.query, w2.db, w2.offsets) == str(g["c2_inputs_sha256"])
    sub = w2.scheme.as_array()
    sc, _, _ = oracle.db_scalar(w2.query, w2.db, w2.offsets, sub, 11, 1)
    assert (sc == g["c2_scalar"]).all()
    prof, bias = oracle.build_profile(w2.query, sub, 16)
    for kern in ("scan", "lazyf"):
        s, _ = oracle.db_striped(kern, prof, bias, w2.db, w2.offsets, 11, 1)
        assert (s == g[f"c2_{kern}_p16"]).all()

    w3 = W.config3(n_pairs=2000)
    assert sha(w3.flat_q, w3.q_off, w3.flat_r, w3.r_off) == str(g["c3_inputs_sha256"])
    sub = w3.scheme.as_array()
    sc, _, _ = oracle.batch_scalar(w3.flat_q, w3.q_off, w3.flat_r, w3.r_off, sub=sub, go=6, ge=1)
    assert (sc == g["c3_scalar"]).all()
    for kern in ("lazyf", "scan"):
        for p in (8, 16):
            s, _, _ = oracle.batch_striped(kern, p, w3.flat_q, w3.q_off, w3.flat_r, w3.r_off,
                                           sub=sub, go=6, ge=1)
            assert (s == g[f"c3_{kern}_p{p}"]).all()

    w4 = W.config4()
    assert sha(w4.query, w4.ref) == str(g["c4_inputs_sha256"])
    sub = w4.scheme.as_array()
    assert oracle.scalar(w4.query, w4.ref, sub, 2, 1)[0] == int(g["c4_scalar"])
    for kern in ("lazyf", "scan"):
        score, _, _, colp = oracle.align_pair(kern, 64, w4.query, w4.ref, sub, 2, 1)
        assert score == int(g[f"c4_{kern}_p64_score"])
        assert (colp == g[f"c4_{kern}_p64_passes"]).all()

    w5 = W.config5(m=8192, n=131_072, block=7_500)
    assert sha(w5.query, w5.ref) == str(g["c5slice_inputs_sha256"])
    sub = w5.scheme.as_array()
    assert oracle.scalar(w5.query, w5.ref, sub, 3, 1)[0] == int(g["c5slice_scalar"])
    assert oracle.align_pair("scan", 64, w5.query, w5.ref, sub, 3, 1)[0] == int(
        g["c5slice_scan_p64"])
