"""The upload path (bm_upload_csc): the row index built chunk by chunk while the
adjacency is copied must be the row index the one-pass build makes (same
offsets, same columns per row), the pulled levels that read it must keep
every maximum, bad input must still be rejected, and pageable host buffers
(copied through the pinned staging ring) must arrive intact."""
import numpy as np
import pytest

import paper_1303_1379_b200 as bm

pytestmark = pytest.mark.gpu


def _transpose(g):
    """The row index of g, computed on the host: offsets and each row's columns sorted."""
    deg = np.diff(g.cxadj)
    cols = np.repeat(np.arange(g.nc, dtype=np.int64), deg)
    rows = g.cadj.astype(np.int64)
    order = np.lexsort((cols, rows))
    roffs = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=g.nr))]).astype(np.uint32)
    return roffs, cols[order].astype(np.int32)


def _canonical(roffs, radj):
    nr = len(roffs) - 1
    rows = np.repeat(np.arange(nr, dtype=np.int64), np.diff(roffs.astype(np.int64)))
    return radj[np.lexsort((radj, rows))]


def _graphs():
    empty_rows = bm.generate_random_bipartite(30000, 50000, 3.0, 12)  # many rows without an edge
    return [bm.generate_random_bipartite(200000, 150000, 6.0, 11), bm.generate_rmat(14, 8.0, 5), empty_rows,
            bm.generate_banded(40000, 3, 0.1, 6)[0], bm.generate_planted(60000, 8.0, 3)]


@pytest.mark.parametrize("chunk", ["4096", "100000", None], ids=["chunk4k", "chunk100k", "chunk_default"])
def test_prebuilt_row_index_equals_one_pass(oracle, monkeypatch, chunk):
    eng = bm.Engine(0)
    if chunk:
        monkeypatch.setenv("BM_UPLOAD_CHUNK", chunk)
    for g in _graphs():
        want_offs, want_cols = _transpose(g)
        monkeypatch.setenv("BM_PREBUILD", "0")
        eng.upload(g, force=True)
        with pytest.raises(ValueError):
            eng.row_index()  # not built yet
        eng.prepare_row_index()
        ro1, ra1 = eng.row_index()
        monkeypatch.setenv("BM_PREBUILD", "1")
        eng.upload(g, force=True)
        ro2, ra2 = eng.row_index()  # built with the upload
        np.testing.assert_array_equal(ro1, want_offs)
        np.testing.assert_array_equal(ro2, want_offs)
        np.testing.assert_array_equal(_canonical(ro1, ra1), want_cols)
        np.testing.assert_array_equal(_canonical(ro2, ra2), want_cols)
        # pulled levels read it (every wide level pulled), then the maximum and a valid matching
        eng.bottom_up = True
        monkeypatch.setenv("BM_BU_FRAC", "0")
        monkeypatch.setenv("BM_SOLO_EDGES", "0")
        m = eng.match(g, bm.cheap_matching(g)).matching
        monkeypatch.delenv("BM_BU_FRAC")
        monkeypatch.delenv("BM_SOLO_EDGES")
        eng.bottom_up = "auto"
        assert bm.cardinality(m) == oracle.maximum(g), g.name
        assert oracle.validate(g, m.rmatch, m.cmatch) == 0
    eng.close()


def test_prebuild_rejects_bad_input(monkeypatch):
    """Out-of-range rows and broken offsets fail the upload with the reference's
    invalid_argument even while the chunks are being bucketed; the handle stays usable."""
    monkeypatch.setenv("BM_PREBUILD", "1")
    monkeypatch.setenv("BM_UPLOAD_CHUNK", "5000")
    eng = bm.Engine(0)
    g = bm.generate_random_bipartite(20000, 15000, 5.0, 77)
    bad = g.cadj.copy()
    bad[len(bad) // 2] = g.nr
    with pytest.raises(ValueError):
        eng.upload(bm.BipartiteCsr(g.nc, g.nr, g.cxadj.copy(), bad), force=True)
    bad[len(bad) // 2] = -5
    with pytest.raises(ValueError):
        eng.upload(bm.BipartiteCsr(g.nc, g.nr, g.cxadj.copy(), bad), force=True)
    cx = g.cxadj.copy()
    cx[100] = cx[101] + 3  # not non-decreasing
    with pytest.raises(ValueError):
        eng.upload(bm.BipartiteCsr(g.nc, g.nr, cx, g.cadj.copy()), force=True)
    eng.upload(g, force=True)
    ro, ra = eng.row_index()
    want_offs, want_cols = _transpose(g)
    np.testing.assert_array_equal(ro, want_offs)
    np.testing.assert_array_equal(_canonical(ro, ra), want_cols)
    eng.close()


def test_pageable_and_pinned_buffers_agree(oracle):
    """Above 8 MB a pageable host buffer goes through the pinned staging ring
    (both directions); the same graph from pinned buffers must give the same
    cardinality, and every downloaded array must match the host's copy."""
    torch = pytest.importorskip("torch")
    g = bm.generate_random_bipartite(1 << 21, 1 << 21, 5.0, 7)  # adjacency ~42 MB, rows 8 MB
    assert g.cadj.nbytes > (8 << 20)
    eng = bm.Engine(0)
    eng.upload(g, force=True)
    back = eng.download_graph()
    np.testing.assert_array_equal(back.cxadj, g.cxadj)
    np.testing.assert_array_equal(back.cadj, g.cadj)
    init = bm.cheap_matching(g)
    m1 = eng.match(g, init).matching
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    gp = bm.BipartiteCsr(g.nc, g.nr, pin(g.cxadj), pin(g.cadj), g.name)
    ip = bm.MatchingState(pin(init.rmatch), pin(init.cmatch))
    eng.upload(gp, force=True)
    m2 = eng.match(gp, ip).matching
    want = oracle.maximum(g)
    assert bm.cardinality(m1) == bm.cardinality(m2) == want
    for m in (m1, m2):
        assert oracle.validate(g, m.rmatch, m.cmatch) == 0
    eng.close()
