"""Graph files on the host (include/bmatch_b200_io.h): CPU tests, plus one GPU
test that runs a file through to the maximum matching.

Matrix Market ingest must reproduce read_matrix_market (matrix_market.cpp:
29-99) exactly: the same CSC for every accepted text, the same ParseError
line and message for every rejected one. It is pinned three ways:
  * golden outcomes of the reference reader (tests/golden/mm_cases.json, made
    by tests/golden/make_mm_golden.py from oracle/_ref);
  * the same texts parsed with tiny chunks, so chunk boundaries fall on every
    line (the parallel path must not change any answer or line number);
  * a live differential run against oracle/_ref on fresh seeds, where it exists.
write_matrix_market output must be byte-identical to the reference's.
"""
import base64
import json
import os
import random

import numpy as np
import pytest

import paper_1303_1379_b200 as bm
from mm_cases import make_case

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "mm_cases.json")))


def _check_outcome(text: bytes, rec: dict):
    if rec["ok"]:
        g = bm.read_matrix_market(text)
        assert (g.nc, g.nr) == (rec["nc"], rec["nr"])
        assert g.cxadj.tolist() == rec["cxadj"]
        assert g.cadj.tolist() == rec["cadj"]
        bm.check_csr(g)
    elif rec["kind"] == "parse":
        with pytest.raises(bm.ParseError) as ei:
            bm.read_matrix_market(text)
        assert ei.value.line == rec["line"], text
        assert str(ei.value) == rec["message"], text
    else:
        # from_edge_list's out_of_range / the reference's length_error on a
        # negative entry count: an argument error, never a ParseError.
        with pytest.raises(ValueError) as ei:
            bm.read_matrix_market(text)
        assert not isinstance(ei.value, bm.ParseError)
        if rec["message"].startswith("edge "):
            assert rec["message"] in str(ei.value)


@pytest.mark.parametrize("chunk", [None, "1", "17"])
def test_matrix_market_matches_reference_golden(chunk, monkeypatch):
    if chunk:
        monkeypatch.setenv("BM_MM_CHUNK", chunk)
    for rec in GOLD["read"]:
        _check_outcome(base64.b64decode(rec["text"]), rec)


def test_matrix_market_reference_kats():
    """The reference's own tests (test_csr_graph.cpp:42-112)."""
    g = bm.read_matrix_market("%%MatrixMarket matrix coordinate pattern general\n2 2 3\n1 1\n2 1\n2 2\n")
    assert (g.nc, g.nr, g.cxadj.tolist(), g.cadj.tolist()) == (2, 2, [0, 2, 3], [0, 1, 1])
    g = bm.read_matrix_market("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 3.5\n2 1 -1.0\n")
    assert (g.cxadj.tolist(), g.cadj.tolist()) == ([0, 2, 3], [0, 1, 0])
    with pytest.raises(bm.ParseError, match="entry count mismatch"):
        bm.read_matrix_market("%%MatrixMarket matrix coordinate pattern general\n1 1 1\n")
    with pytest.raises(bm.ParseError):
        bm.read_matrix_market("%%MatrixMarket matrix array real general\n")
    with pytest.raises(bm.ParseError) as ei:
        bm.read_matrix_market("not a header\n")
    assert ei.value.line == 1
    with pytest.raises(bm.ParseError) as ei:
        bm.read_matrix_market("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n3 1\n")
    assert ei.value.line == 3
    with pytest.raises(bm.ParseError, match="entry count mismatch"):
        bm.read_matrix_market("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n2 2\n")


def test_matrix_market_write_matches_reference_bytes(tmp_path):
    for rec in GOLD["write"]:
        g = bm.generate_random_bipartite(rec["nc"], rec["nr"], rec["deg"], rec["seed"])
        p = tmp_path / "g.mtx"
        bm.write_matrix_market(g, str(p))
        assert p.read_bytes() == base64.b64decode(rec["text"])


def test_matrix_market_large_round_trip_and_late_errors(tmp_path, monkeypatch):
    g = bm.generate_random_bipartite(200000, 150000, 6.0, 7)
    p = tmp_path / "big.mtx"
    bm.write_matrix_market(g, str(p), threads=4)
    for chunk, threads in [(None, 0), ("100000", 16), ("4096", 3)]:
        if chunk:
            monkeypatch.setenv("BM_MM_CHUNK", chunk)
        back = bm.load_matrix_market(str(p), threads=threads)
        assert back.name == "big"
        assert (back.nc, back.nr) == (g.nc, g.nr)
        assert np.array_equal(back.cxadj, g.cxadj) and np.array_equal(back.cadj, g.cadj)
    # Corrupt one entry deep in the file: the error names exactly its line.
    lines = p.read_bytes().split(b"\n")
    k = 2 + 3 * len(lines) // 4  # 1-based line number of the line we break
    lines[k - 1] = b"1 0"
    bad = tmp_path / "bad.mtx"
    bad.write_bytes(b"\n".join(lines))
    with pytest.raises(bm.ParseError) as ei:
        bm.load_matrix_market(str(bad))
    assert ei.value.line == k
    assert "column index 0 outside" in str(ei.value)
    # Extra data after the declared entries, after a run of comments.
    extra = tmp_path / "extra.mtx"
    extra.write_bytes(p.read_bytes() + b"% c\n\n  \n5 5\n")
    with pytest.raises(bm.ParseError) as ei:
        bm.load_matrix_market(str(extra))
    assert ei.value.line == len(lines) + 3  # the text ended with '\n'
    assert "data after the declared" in str(ei.value)


def test_matrix_market_live_differential_against_reference():
    try:
        from oracle import Reference
        ref = Reference()
    except ImportError:
        pytest.skip("oracle/_ref not built (the reference tree is absent)")
    rng = random.Random(5)
    for seed in range(50000, 50400):
        text = make_case(seed)
        r = ref.read_matrix_market(text)
        if r[0] == "ok":
            rec = dict(ok=True, nc=r[1], nr=r[2], cxadj=r[3].tolist(), cadj=r[4].tolist())
        elif r[0] == "parse":
            rec = dict(ok=False, kind="parse", line=r[1], message=r[2])
        else:
            rec = dict(ok=False, kind="error", message=r[1])
        _check_outcome(text, rec)
    for _ in range(5):
        nc, nr = rng.randint(0, 500), rng.randint(0, 500)
        g = bm.generate_random_bipartite(nc, nr, rng.uniform(0.5, 6), rng.randint(0, 99))
        assert bm.read_matrix_market(ref.write_matrix_market(g)).cadj.tolist() == g.cadj.tolist()


def test_file_errors(tmp_path):
    with pytest.raises(OSError):
        bm.load_matrix_market(str(tmp_path / "missing.mtx"))
    with pytest.raises(OSError):
        bm.load_csc(str(tmp_path / "missing.bcsc"))
    with pytest.raises(bm.ParseError) as ei:
        empty = tmp_path / "empty.mtx"
        empty.write_bytes(b"")
        bm.load_matrix_market(str(empty))
    assert ei.value.line == 1


def test_binary_csc_round_trip_and_corruption(tmp_path):
    for g in [bm.generate_random_bipartite(0, 0, 1.0, 1), bm.generate_random_bipartite(3000, 2000, 5.0, 2),
              bm.generate_rmat(12, 8.0, 3)]:
        p = tmp_path / "g.bcsc"
        bm.save_csc(g, str(p), threads=4)
        back = bm.load_csc(str(p))
        assert (back.nc, back.nr) == (g.nc, g.nr)
        assert np.array_equal(back.cxadj, g.cxadj) and np.array_equal(back.cadj, g.cadj)
        assert bm.csc_digest(back) == bm.csc_digest(g)
    raw = bytearray(p.read_bytes())
    raw[-5] ^= 0x10  # flip one bit of cadj
    p.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="checksum"):
        bm.load_csc(str(p))
    p.write_bytes(bytes(raw[:-4]))
    with pytest.raises(ValueError, match="file size"):
        bm.load_csc(str(p))
    p.write_bytes(b"not a csc file at all, padded to forty bytes!!")
    with pytest.raises(ValueError, match="BMCSC001"):
        bm.load_csc(str(p))


def test_parallel_check_csc_matches_serial_messages():
    g = bm.generate_random_bipartite(200000, 1000, 4.0, 9)
    bm.check_csr(g)
    bad = bm.BipartiteCsr(g.nc, g.nr, g.cxadj.copy(), g.cadj.copy())
    c = 150000
    j = int(bad.cxadj[c])
    bad.cadj[j] = bad.cadj[j + 1]  # column c no longer strictly ascending
    with pytest.raises(ValueError, match=f"column {c} slice is not strictly ascending"):
        bm.check_csr(bad)
    bad.cadj[int(bad.cxadj[90000])] = 5000  # an earlier column with an out-of-range row wins
    with pytest.raises(ValueError, match="row index out of range in column 90000"):
        bm.check_csr(bad)


@pytest.mark.gpu
def test_files_to_maximum_matching_on_gpu(tmp_path):
    """File in, matching out: a Matrix Market file and its BMCSC001 copy load to
    the same graph, and the engine finds the reference's known maximum on it
    (C1: generate_random_bipartite(100000, 100000, 8.0, 1) -> 99,961)."""
    g = bm.generate_random_bipartite(100000, 100000, 8.0, 1)
    mtx, bcsc = tmp_path / "c1.mtx", tmp_path / "c1.bcsc"
    bm.write_matrix_market(g, str(mtx))
    h = bm.load_matrix_market(str(mtx))
    bm.save_csc(h, str(bcsc))
    for gg in (h, bm.load_csc(str(bcsc))):
        assert np.array_equal(gg.cadj, g.cadj)
        res = bm.apfb(gg, bm.cheap_matching(gg), None, None, bm.BfsKernel.GpubfsWr)
        assert bm.cardinality(res.matching) == 99961
