"""CPU-only tests of the host side: the C-ABI library surface, generators and
CSC helpers, and the Python mirror of the reference interface (registry,
errors). No compute call needs a GPU here; device entry points are checked
to fail loudly (no CPU fallback)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_1303_1379_b200 as bm
from paper_1303_1379_b200 import _lib
from conftest import fork_graph

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


# ---- C ABI ------------------------------------------------------------------------
def test_library_exports_every_declared_symbol():
    names = _lib.declared_symbols()
    assert "bm_match" in names and "bm_upload_csc" in names and "bm_gen_uniform" in names
    raw = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in names if not hasattr(raw, n)]
    assert not missing, missing
    assert _lib.lib.bm_abi_version() == 1


def test_status_strings():
    for s in range(7):
        assert _lib.lib.bm_status_string(s)


def test_no_cpu_fallback_without_gpu():
    """Without a usable device the engine refuses to run (BM_ERR_CUDA), it
    never silently computes on the CPU."""
    if _lib.lib.bm_device_count() > 0:
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    st = _lib.lib.bm_create(0, C.byref(h))
    assert st == _lib.BM_ERR_CUDA
    assert b"no CUDA device" in _lib.lib.bm_last_error()
    with pytest.raises(bm.CudaError):
        bm.Engine(0)
    # the multi-GPU engine refuses as well
    from paper_1303_1379_b200 import partition
    st = partition.lib.bm_mg_create(0, 0, 2, 1, C.byref(h))
    assert st == _lib.BM_ERR_CUDA
    assert partition.lib.bm_mg_create(0, 3, 2, 1, C.byref(h)) == _lib.BM_ERR_INVALID_ARG  # rank out of range
    assert partition.lib.bm_mg_create(0, 0, 9, 1, C.byref(h)) == _lib.BM_ERR_INVALID_ARG  # world > 8


def test_null_handle_errors():
    assert _lib.lib.bm_upload_csc(None, 1, 1, None, None) == _lib.BM_ERR_INVALID_ARG
    assert _lib.lib.bm_destroy(None) == _lib.BM_OK


# ---- generators ---------------------------------------------------------------------
def test_uniform_generator_matches_reference_digests():
    """generate_random_bipartite is bit-identical to the reference (csr_graph.cpp:92-112)."""
    with open(os.path.join(GOLDEN, "known_answers.json")) as f:
        ka = json.load(f)
    for key in ["uniform/100000/8.0/1", "uniform/200000/6.0/4242", "uniform/1000000/8.0/1"]:
        _, n, d, s = key.split("/")
        g = bm.generate_random_bipartite(int(n), int(n), float(d), int(s))
        assert g.num_edges() == ka[key]["edges"]
        assert bm.csc_digest(g) == int(ka[key]["digest"])
    # thread count does not change the result
    a = bm.generate_random_bipartite(50000, 40000, 5.0, 99, threads=1)
    b = bm.generate_random_bipartite(50000, 40000, 5.0, 99, threads=7)
    assert np.array_equal(a.cxadj, b.cxadj) and np.array_equal(a.cadj, b.cadj)


def test_generators_are_valid_csc_and_deterministic():
    gs = [bm.generate_planted(20000, 16.0, 2024), bm.generate_rmat(14, 16.0, 2024),
          bm.generate_banded(30000, 3, 0.05, 12345)[0], bm.generate_random_bipartite(3000, 5000, 4.0, 1)]
    for g in gs:
        bm.check_csr(g)
    for f in [lambda t: bm.generate_planted(20000, 16.0, 7, threads=t), lambda t: bm.generate_rmat(12, 8.0, 3, threads=t),
              lambda t: bm.generate_banded(20000, 3, 0.05, 5, threads=t)[0]]:
        a, b = f(1), f(5)
        assert np.array_equal(a.cxadj, b.cxadj) and np.array_equal(a.cadj, b.cadj)


def test_planted_contains_a_perfect_matching(oracle):
    g = bm.generate_planted(5000, 8.0, 11)
    assert oracle.maximum(g) == 5000


def test_banded_maximum_is_live_rows(oracle):
    g, live = bm.generate_banded(20000, 3, 0.05, 12345)
    assert 0.9 * 20000 < live < 20000
    assert oracle.maximum(g) == live
    assert (np.diff(g.cxadj) <= 3).all()


def test_rmat_is_skewed():
    g = bm.generate_rmat(16, 16.0, 2024)
    deg = np.diff(g.cxadj)
    assert deg.max() > 50 * max(deg.mean(), 1)
    assert (deg == 0).mean() > 0.2


def test_known_answers_fixture_matches_generators():
    with open(os.path.join(GOLDEN, "known_answers.json")) as f:
        ka = json.load(f)
    g = bm.generate_planted(1_000_000, 16.0, 2024)
    assert bm.csc_digest(g) == int(ka["planted/1000000/16/2024"]["digest"])
    assert ka["planted/1000000/16/2024"]["maximum"] == 1_000_000
    g, live = bm.generate_banded(1_000_000, 3, 0.05, 12345)
    assert bm.csc_digest(g) == int(ka["banded/1000000/3/0.05/12345"]["digest"])
    assert ka["banded/1000000/3/0.05/12345"]["maximum"] == live


def test_check_csr_rejects_bad_graphs():
    """csr_graph.cpp:45-64"""
    ok = bm.BipartiteCsr(2, 3, np.array([0, 1, 3]), np.array([2, 0, 1]))
    bm.check_csr(ok)
    with pytest.raises(ValueError, match="not strictly ascending"):
        bm.check_csr(bm.BipartiteCsr(2, 3, np.array([0, 1, 3]), np.array([2, 1, 0])))
    with pytest.raises(ValueError, match="out of range"):
        bm.check_csr(bm.BipartiteCsr(2, 3, np.array([0, 1, 3]), np.array([2, 0, 3])))
    with pytest.raises(ValueError, match="decreases"):
        bm.check_csr(bm.BipartiteCsr(2, 3, np.array([0, 2, 1]), np.array([0])))


def test_from_edge_list():
    """csr_graph.cpp:10-43: sorted, de-duplicated; out_of_range names the edge."""
    g = bm.BipartiteCsr.from_edge_list(3, 4, [(2, 1), (0, 3), (0, 1), (2, 1)])
    assert g.cxadj.tolist() == [0, 2, 2, 3] and g.cadj.tolist() == [1, 3, 1]
    with pytest.raises(IndexError, match="edge 1"):
        bm.BipartiteCsr.from_edge_list(2, 2, [(0, 0), (2, 0)])


# ---- registry / interface mirror --------------------------------------------------------
def test_registry_ids_and_lookup():
    ids = bm.algorithm_ids()
    assert ids == ["apfb-gpubfs-b200", "apfb-wr-b200", "apsb-gpubfs-b200", "apsb-wr-b200"]
    for i in ids:
        assert callable(bm.make_algorithm(i))
    assert bm.make_algorithm("nope") is None
    assert bm.make_algorithm("apfb-wr") is None  # only the -b200 ids live here


def test_registered_ids_are_consulted_first():
    """algorithms.cpp:64-67, 95-97 (and the broken-for-tests fault injection, test_cli.cpp:205-224)."""
    calls = []

    def broken(g, init, schedule=None):
        calls.append(1)
        return bm.AlgorithmResult(bm.MatchingState.unmatched(g.nc, g.nr))

    bm.register_algorithm("apfb-wr-b200", broken)
    try:
        res = bm.make_algorithm("apfb-wr-b200")(fork_graph(), bm.cheap_matching(fork_graph()))
        assert calls == [1] and bm.cardinality(res.matching) == 0
    finally:
        bm.api._EXTRA.pop("apfb-wr-b200")
    assert bm.make_algorithm("apfb-wr-b200") is not broken


def test_improved_requires_wr_kernel():
    """gpu_match.cpp:272-274 — raised before any device work."""
    with pytest.raises(bm.LogicError):
        bm.apsb(fork_graph(), bm.cheap_matching(fork_graph()), None, None, bm.BfsKernel.Gpubfs, True)


def test_cheap_matching_is_maximal(oracle):
    """test_matching.cpp:35-50"""
    g = bm.generate_random_bipartite(3000, 2500, 3.0, 42)
    m = bm.cheap_matching(g)
    assert oracle.validate(g, m.rmatch, m.cmatch) == 0
    for c in range(g.nc):
        if m.cmatch[c] < 0:
            assert (m.rmatch[g.column(c)] >= 0).all()
    r, c = oracle.cheap_matching(g)
    assert np.array_equal(r, m.rmatch) and np.array_equal(c, m.cmatch)
