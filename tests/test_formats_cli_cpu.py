"""Formats, runner validation and CLI usage errors (no device work)."""

from __future__ import annotations

import io

import numpy as np
import pytest

from paper_1909_00899_b200 import cli, formats, runner
from paper_1909_00899_b200.scoring import Alphabet, ScoringScheme


def test_parse_fasta_records_case_blank_crlf():
    recs = formats.parse_fasta(b">a desc here\r\nacgt\r\n\r\nTT\n>b\nG\n")
    assert [(r.id, r.description, r.sequence) for r in recs] == [
        ("a", "desc here", "ACGTTT"), ("b", "", "G")]
    assert formats.parse_fasta(io.StringIO(">x\nAC\n"))[0].sequence == "AC"


@pytest.mark.parametrize("bad", [b"ACGT\n>a\nA\n", b">a\n\n>b\nA\n", b">\nACGT\n",
                                 b">a\nAC\xff\n"])
def test_parse_fasta_errors(bad):
    with pytest.raises(formats.MalformedFasta):
        formats.parse_fasta(bad)


def test_parse_fasta_alphabet_check():
    with pytest.raises(formats.MalformedFasta):
        formats.parse_fasta(b">a\nACGX\n", Alphabet.dna())
    assert formats.parse_fasta(b">a\nacgn\n", Alphabet.dna())[0].sequence == "ACGN"


def test_parse_matrix_and_errors():
    alph, rows = formats.parse_matrix("A B\n1 -1\n-1 2\n")
    assert alph.symbols == "AB" and rows == ((1, -1), (-1, 2))
    for bad in ("", "AB C\n1 2\n3 4\n", "A A\n1 1\n1 1\n", "A B\n1 2\n", "A B\n1 2\n3\n",
                "A B\n1 x\n3 4\n"):
        with pytest.raises(formats.MalformedMatrix):
            formats.parse_matrix(bad)


def test_encode_records_and_packed_db():
    recs = formats.parse_fasta(">a\nACGT\n>b\nGG\n>c\nTTTAC\n")
    codes, off = formats.encode_records(recs, Alphabet("ACGT"))
    assert codes.tolist() == [0, 1, 2, 3, 2, 2, 3, 3, 3, 0, 1] and off.tolist() == [0, 4, 6, 11]
    _, packed = formats.load_fasta_db(">a\nACGT\n>b\nGG\n>c\nTTTAC\n", Alphabet("ACGT"),
                                      pin=False)
    assert packed.ids.tolist() == [2, 0, 1]  # length-descending physical order
    assert packed.length.tolist() == [5, 4, 2]
    assert packed.codes[:5].tolist() == [3, 3, 3, 0, 1]


def test_generate_pairs_is_the_reference_generator():
    # draw order (query len, target len, query, target) and wildcard exclusion
    a = runner.generate_pairs(5, 3, 9, 42, Alphabet.dna())
    rng = np.random.default_rng(42)
    for q, t in a:
        lq = int(rng.integers(3, 10))
        lt = int(rng.integers(3, 10))
        assert q == "".join("ACGT"[i] for i in rng.integers(0, 4, lq))
        assert t == "".join("ACGT"[i] for i in rng.integers(0, 4, lt))
    assert runner.generate_pairs(5, 3, 9, 42, Alphabet.dna()) == a
    with pytest.raises(ValueError):
        runner.generate_pairs(-1, 1, 2, 0, Alphabet.dna())


def test_runner_validation_returns_1(capsys):
    assert runner.run(runner.RunConfig(kernel="bogus", random_count=1)) == 1
    assert runner.run(runner.RunConfig(lanes=3, random_count=1)) == 1
    assert runner.run(runner.RunConfig(query_path="/nonexistent.fa",
                                       target_path="/nonexistent.fa")) == 1
    assert "error:" in capsys.readouterr().err


@pytest.mark.parametrize("argv", [["--random", "3", "--query", "q.fa"], [], ["--random", "-1"],
                                  ["--random", "2", "--bench", "0"],
                                  ["--random", "2", "--len-min", "5", "--len-max", "2"],
                                  ["--random", "2", "--lanes", "3"]])
def test_cli_usage_errors_exit_2(argv):
    with pytest.raises(SystemExit) as e:
        cli.main(argv)
    assert e.value.code == 2


def test_scheme_from_matrix_file(tmp_path):
    f = tmp_path / "m.txt"
    f.write_text("A C\n2 -3\n-3 2\n")
    alph, sch = runner._build_scheme(runner.RunConfig(matrix_path=str(f), gap_open=5,
                                                      gap_extend=2))
    assert alph.symbols == "AC" and sch == ScoringScheme(((2, -3), (-3, 2)), 5, 2)


def test_packed_db_save_load_roundtrip(tmp_path):
    from paper_1909_00899_b200 import search, workloads as W

    w = W.config2(n_targets=500)
    packed = search.pack(w.db, w.offsets, pin=False)
    search.save_packed(str(tmp_path / "db"), packed, alphabet="stand-in")
    back, meta = search.load_packed(str(tmp_path / "db"), pin=False)
    assert meta["n"] == 500 and meta["residues"] == int(w.offsets[-1])
    for name in search.PACKED_FILES:
        assert (getattr(back, name).numpy() == getattr(packed, name).numpy()).all(), name
    (tmp_path / "db" / "meta.json").write_text('{"format": "other"}')
    import pytest

    with pytest.raises(ValueError):
        search.load_packed(str(tmp_path / "db"), pin=False)


def test_shard_pairs_partition():
    from paper_1909_00899_b200 import search

    for n in (0, 1, 7, 1 << 20):
        for world in (1, 2, 3, 8):
            parts = [search.shard_pairs(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def _reference_formats():
    import importlib
    import os
    import sys

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline",
                       "_ref")
    if not os.path.isdir(os.path.join(ref, "swscan")):
        pytest.skip("reference package not installed in baseline/_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/swscan_numba_cache")
    return importlib.import_module("swscan.formats"), importlib.import_module("swscan.scoring")


def _random_fasta(rng) -> bytes:
    pieces = [b">", b"> ", b">id", b">id desc", b">a  b c ", b"\n", b"\r\n", b"\r", b"\x0b",
              b"\x0c", b"\x1c", b"  ", b"\t", b"\x1f", b"ACGT", b"acgt", b"N", b"AC GT", b"X",
              b"-", b"*", b"GATTACA", b"gg", b">q1", b">q2 x"]
    k = int(rng.integers(0, 14))
    return b"".join(pieces[int(i)] for i in rng.integers(0, len(pieces), k))


def test_read_fasta_slices_agree(monkeypatch):
    """The threaded byte passes (buffer cut at line breaks) give the single-slice result."""
    rng = np.random.default_rng(0x511CE)
    data = b"".join(_random_fasta(rng) for _ in range(3000)) + b"\n>z\nACGT\n"
    data = b">a\n" + data.replace(b">\n", b">x\n").replace(b"> \n", b">y\n")
    try:
        one = formats.read_fasta(data, None, threads=1)
        want = (one.ids, one.descriptions, one.codes.tolist(), one.offsets.tolist())
    except formats.MalformedFasta as e:
        want = str(e)
    monkeypatch.setattr(formats, "_MIN_SPLIT", 1)
    for t in (2, 3, 7, 16):
        try:
            b = formats.read_fasta(data, None, threads=t)
            got = (b.ids, b.descriptions, b.codes.tolist(), b.offsets.tolist())
        except formats.MalformedFasta as e:
            got = str(e)
        assert got == want, t


def test_parse_fasta_differential_vs_reference():
    """The byte-level ingester against the reference's line parser on 4,000 random
    inputs built from FASTA's corner cases: identical records, or the same
    MalformedFasta message (the first problem the reference meets)."""
    ref_formats, ref_scoring = _reference_formats()
    rng = np.random.default_rng(0xFA57A)
    for i in range(4000):
        data = _random_fasta(rng)
        for alph in (None, "dna"):
            a_ref = ref_scoring.Alphabet.dna() if alph else None
            a_new = Alphabet.dna() if alph else None
            try:
                want = [(r.id, r.description, r.sequence) for r in
                        ref_formats.parse_fasta(data, a_ref)]
            except ref_formats.MalformedFasta as e:
                want = ("error", str(e))
            try:
                got = [(r.id, r.description, r.sequence) for r in formats.parse_fasta(data, a_new)]
            except formats.MalformedFasta as e:
                got = ("error", str(e))
            assert got == want, (i, data, alph)
            if alph and not isinstance(want, tuple):
                b = formats.read_fasta(data, a_new)
                codes = [list(a_new.lut()[np.frombuffer(s.encode(), np.uint8)]) for _, _, s in want]
                assert [b.codes[b.offsets[j]:b.offsets[j + 1]].tolist() for j in range(len(b))] == codes
    # non-ASCII bytes: same error class and message as the reference's decode
    for bad in (b">a\nAC\xff\n", b"\x80"):
        with pytest.raises(ref_formats.MalformedFasta) as e1:
            ref_formats.parse_fasta(bad)
        with pytest.raises(formats.MalformedFasta) as e2:
            formats.parse_fasta(bad)
        assert str(e1.value) == str(e2.value)


def test_read_fasta_million_records_is_vectorised():
    """1,000,000 records (~30M residues) parse and encode in a few seconds."""
    import time

    rng = np.random.default_rng(5)
    lens = rng.integers(10, 50, 1_000_000)
    body = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, int(lens.sum()))]
    lines = []
    o = 0
    for i, ln in enumerate(lens[:1000]):  # a hand-made prefix for the content check
        lines.append(b">r%d d\n" % i + body[o:o + ln].tobytes() + b"\n")
        o += ln
    # the rest assembled in bulk (header + sequence per record)
    hdr = np.char.add(np.char.add(">r", np.arange(1000, 1_000_000).astype(str)), " d\n")
    seqs = np.split(body[o:], np.cumsum(lens[1000:])[:-1])
    rest = b"".join(h.encode() + s.tobytes() + b"\n" for h, s in zip(hdr, seqs))
    data = b"".join(lines) + rest
    t0 = time.perf_counter()
    b = formats.read_fasta(data, Alphabet("ACGT"))
    dt = time.perf_counter() - t0
    assert len(b) == 1_000_000 and (b.lengths == lens).all()
    assert b.ids[12345] == "r12345" and b.descriptions[7] == "d"
    lut = Alphabet("ACGT").lut()
    assert (b.codes[: lens[0]] == lut[body[: lens[0]]]).all()
    assert (b.codes[-lens[-1]:] == lut[body[-lens[-1]:]]).all()
    assert dt < 20.0, dt


def test_pack_2bit_roundtrip():
    from paper_1909_00899_b200.formats import pack_2bit, unpack_2bit

    rng = np.random.default_rng(5)
    for n in (0, 1, 2, 3, 4, 5, 31, 32, 33, 4097):
        c = rng.integers(0, 4, n).astype(np.uint8)
        p = pack_2bit(c)
        assert p.dtype == np.uint8 and p.size == (n + 3) // 4
        assert (unpack_2bit(p, n) == c).all()
    assert pack_2bit(np.array([1, 2, 3, 0, 3], np.uint8)).tolist() == [1 | 2 << 2 | 3 << 4, 3]
    with pytest.raises(ValueError):
        pack_2bit(np.array([0, 4], np.uint8))

