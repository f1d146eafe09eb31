"""Pins the C oracle (oracle/bm_oracle.c) to the reference before it is
trusted as the GPU checker:
  * the reference's own known-answer tests (proj/tests/test_gpu_match.cpp,
    test_matching.cpp), restated with their file:line;
  * golden fixtures produced by the reference itself (tests/golden/, made by
    make_golden.py from oracle/_ref = the reference sources compiled
    unmodified): 1004-instance acceptance corpus with Serial-schedule counters
    of all 8 registry configs, and single-kernel traces.
Runs on CPU only.
"""
import json
import os

import numpy as np
import pytest

import paper_1303_1379_b200 as bm
from conftest import fork_graph, fork_partial_matching

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CONFIGS = {  # id -> (shortest, kernel, improved, grid)  algorithms.cpp:19-27
    "apfb-gpubfs": (0, 0, 0), "apfb-wr": (0, 1, 0), "apsb-gpubfs": (1, 0, 0), "apsb-wr": (1, 1, 1)}


def _arr(x):
    return np.asarray(x, dtype=np.int32)


# ---- reference KATs -----------------------------------------------------------
def test_init_arrays(oracle):
    """test_gpu_match.cpp:39-49"""
    out = np.zeros(3, np.int32)
    oracle.lib.or_init_bfs_array(3, np.ctypeslib.as_ctypes(_arr([-1, 3, -1])), 2, np.ctypeslib.as_ctypes(out))
    assert out.tolist() == [2, 1, 2]
    out = np.zeros(3, np.int32)
    oracle.lib.or_init_root(3, np.ctypeslib.as_ctypes(_arr([5, -1, -1])), np.ctypeslib.as_ctypes(out))
    assert out.tolist() == [0, 1, 2]


def _level(oracle, g, m, level, bfs, pred, rmatch, root=None, improved=0, tot=8):
    import ctypes as C
    flags = np.array([0, 0], np.int32)
    G = C.byref(oracle.graph(g))
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    if root is None:
        n = oracle.lib.or_gpubfs(G, tot, level, 2, p(bfs), p(pred), p(rmatch), p(flags))
    else:
        n = oracle.lib.or_gpubfs_wr(G, tot, level, 2, improved, p(bfs), p(pred), p(root), p(rmatch), p(flags))
    return n, flags


def test_fork_gpubfs_trace(oracle):
    """test_gpu_match.cpp:51-71"""
    g, m = fork_graph(), fork_partial_matching()
    bfs, pred, rm = _arr([2, 1]), np.full(3, -1, np.int32), m.rmatch.copy()
    _, f = _level(oracle, g, m, 2, bfs, pred, rm)
    assert bfs.tolist() == [2, 3] and pred[0] == 0 and f.tolist() == [1, 0] and rm.tolist() == [1, -1, -1]
    _, f = _level(oracle, g, m, 3, bfs, pred, rm)
    assert rm.tolist() == [1, -2, -2] and pred.tolist() == [0, 1, 1] and f.tolist() == [0, 1]


def test_fork_improved_root_encoding(oracle):
    """test_gpu_match.cpp:111-129: bfs[0] == -2 (the later endpoint r2 wins)."""
    g, m = fork_graph(), fork_partial_matching()
    bfs, pred, rm, root = _arr([2, 1]), np.full(3, -1, np.int32), m.rmatch.copy(), _arr([0, 0])
    _level(oracle, g, m, 2, bfs, pred, rm, root=root, improved=1)
    assert bfs.tolist() == [2, 3] and root.tolist() == [0, 0]
    _, f = _level(oracle, g, m, 3, bfs, pred, rm, root=root, improved=1)
    assert bfs[0] == -2 and rm.tolist() == [1, -2, -2] and f[1] == 1


def test_fork_alternate_and_fix(oracle):
    """test_gpu_match.cpp:154-173"""
    import ctypes as C
    g = fork_graph()
    rm, cm, pred = _arr([1, -2, -2]), _arr([-1, 0]), _arr([0, 1, 1])
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    walks = oracle.lib.or_alternate(C.byref(oracle.graph(g)), 8, p(pred), p(rm), p(cm))
    assert walks == 2 and cm.tolist() == [0, 1] and rm.tolist() == [0, 1, -2]
    resets = oracle.lib.or_fix_matching(2, 3, p(rm), p(cm))
    assert rm.tolist() == [0, 1, -1] and resets == 1
    assert oracle.validate(g, rm, cm) == 0


def test_alternate_wr_and_length_one(oracle):
    """test_gpu_match.cpp:185-211"""
    import ctypes as C
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    one = bm.BipartiteCsr.from_edge_list(1, 1, [(0, 0)])
    rm, cm = _arr([-2]), _arr([-1])
    oracle.lib.or_alternate(C.byref(oracle.graph(one)), 8, p(_arr([0])), p(rm), p(cm))
    assert rm.tolist() == [0] and cm.tolist() == [0]
    g = fork_graph()
    rm, cm = _arr([1, -2, -2]), _arr([-1, 0])
    walks = oracle.lib.or_alternate_wr(C.byref(oracle.graph(g)), 8, p(_arr([-1, 3])), p(_arr([0, 1, 1])), p(rm),
                                       p(cm))
    assert walks == 1 and cm.tolist() == [0, 1] and rm.tolist() == [0, 1, -2]


def test_fix_rules(oracle):
    """test_gpu_match.cpp:245-272"""
    import ctypes as C
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    rm, cm = _arr([0, 0]), _arr([0])
    oracle.lib.or_fix_matching(1, 2, p(rm), p(cm))
    assert rm.tolist() == [0, -1] and cm.tolist() == [0]
    rm, cm = _arr([-2]), _arr([-1])
    oracle.lib.or_fix_matching(1, 1, p(rm), p(cm))
    assert rm.tolist() == [-1]
    rm, cm = _arr([1]), _arr([0, 0])
    oracle.lib.or_fix_matching(2, 1, p(rm), p(cm))
    assert cm.tolist() == [-1, 0] and rm.tolist() == [1]


def test_driver_kats(oracle):
    """test_gpu_match.cpp:274-306"""
    g = fork_graph()
    r0, c0 = oracle.cheap_matching(g)
    st, r, c, ct = oracle.driver(g, r0, c0, tot=8, kernel=0)
    assert st == 0 and (r >= 0).sum() == 2 and ct["outer_iterations"] == 1
    e = bm.BipartiteCsr.from_edge_list(3, 4, [])
    st, r, c, ct = oracle.driver(e, np.full(4, -1, np.int32), np.full(3, -1, np.int32), tot=8)
    assert ct["outer_iterations"] == 1 and (r == -1).all()
    m = fork_partial_matching()
    st, r, c, ct = oracle.driver(g, m.rmatch, m.cmatch, tot=8, shortest=True, kernel=1, improved=True)
    assert (r >= 0).sum() == 2 and oracle.is_maximum(g, r, c) == 1
    comp = bm.BipartiteCsr.from_edge_list(3, 3, [(a, b) for a in range(3) for b in range(3)])
    r0, c0 = oracle.cheap_matching(comp)
    st, r, c, ct = oracle.driver(comp, r0, c0, tot=8, shortest=True, kernel=0)
    assert ct["outer_iterations"] == 1 and ct["bfs_launches_per_iteration"] == [1]
    assert oracle.driver(g, r0[:3], c0[:2], tot=8, kernel=0, improved=True)[0] == 2  # logic_error


def test_cheap_matching_kats(oracle):
    """test_matching.cpp:12-33 (oracle and the product's host first-fit agree)."""
    g = bm.BipartiteCsr.from_edge_list(2, 2, [(0, 0), (0, 1), (1, 0)])
    r, c = oracle.cheap_matching(g)
    assert c.tolist() == [0, -1] and r.tolist() == [0, -1]
    m = bm.cheap_matching(g)
    assert m.cmatch.tolist() == [0, -1] and m.rmatch.tolist() == [0, -1]
    r, c = oracle.cheap_matching(fork_graph())
    assert c.tolist() == [0, 1] and r.tolist() == [0, 1, -1]


# ---- golden fixtures produced by the reference ------------------------------------
@pytest.fixture(scope="module")
def corpus_golden():
    with open(os.path.join(GOLDEN, "corpus.json")) as f:
        return json.load(f)


def test_corpus_matches_reference(oracle, corpus_golden):
    """Every corpus instance: generator digest, brute force, first-fit and the
    exact Serial-schedule counters of all 8 registry configs (CT grid 256)."""
    import conftest
    graphs = conftest.acceptance_corpus(1000)
    assert len(graphs) == len(corpus_golden) == 1004
    for g, gold in zip(graphs, corpus_golden):
        assert bm.csc_digest(g) == int(gold["digest"]), g.name
        assert oracle.brute_force_maximum(g) == gold["maximum"]
        assert oracle.maximum(g) == gold["maximum"]  # Hopcroft-Karp restatement
        r0, c0 = oracle.cheap_matching(g)
        assert int((r0 >= 0).sum()) == gold["first_fit"]
        for algo, want in gold["runs"].items():
            base, grid = algo[:-3], algo[-2:]
            shortest, kernel, improved = CONFIGS[base]
            tot = 256 if grid == "ct" else max(1, min(g.nc, 65536))
            st, r, c, ct = oracle.driver(g, r0, c0, tot=tot, shortest=shortest, kernel=kernel, improved=improved)
            assert st == 0
            assert int((r >= 0).sum()) == gold["maximum"]
            assert ct == want, (g.name, algo)


def test_kernel_steps_match_reference(oracle):
    """Single-level traces (bfs/pred/root/rmatch/flags/scans) and the ALTERNATE
    and FIX results, exactly as the reference produced them."""
    import ctypes as C
    with open(os.path.join(GOLDEN, "steps.json")) as f:
        cases = json.load(f)
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    for case in cases:
        g = bm.generate_random_bipartite(case["nc"], case["nr"], case["deg"], case["seed"])
        nc, nr = g.nc, g.nr
        r, c = _arr(case["init_rmatch"]), _arr(case["init_cmatch"])
        bfs = np.zeros(nc, np.int32)
        oracle.lib.or_init_bfs_array(nc, p(c), 2, p(bfs))
        root = np.zeros(nc, np.int32)
        oracle.lib.or_init_root(nc, p(c), p(root))
        pred = np.full(nr, -1, np.int32)
        G = C.byref(oracle.graph(g))
        for lv in case["levels"]:
            flags = np.array([0, 0], np.int32)
            if case["wr"]:
                n = oracle.lib.or_gpubfs_wr(G, 64, lv["level"], 2, case["improved"], p(bfs), p(pred), p(root), p(r),
                                            p(flags))
            else:
                n = oracle.lib.or_gpubfs(G, 64, lv["level"], 2, p(bfs), p(pred), p(r), p(flags))
            assert n == lv["scans"]
            assert bfs.tolist() == lv["bfs"] and pred.tolist() == lv["pred"] and r.tolist() == lv["rmatch"]
            if case["wr"]:
                assert root.tolist() == lv["root"]
            assert bool(flags[0]) == bool(lv["flags"][0])
        ra, ca = r.copy(), c.copy()
        if case["improved"]:
            walks = oracle.lib.or_alternate_wr(G, 64, p(bfs), p(pred), p(ra), p(ca))
        else:
            walks = oracle.lib.or_alternate(G, 64, p(pred), p(ra), p(ca))
        assert walks == case["alternate"]["walks"]
        assert ra.tolist() == case["alternate"]["rmatch"] and ca.tolist() == case["alternate"]["cmatch"]
        resets = oracle.lib.or_fix_matching(nc, nr, p(ra), p(ca))
        assert resets == case["fix"]["resets"] and ra.tolist() == case["fix"]["rmatch"]


def test_known_answers_oracle(oracle):
    """Reference cardinalities on larger inputs (known_answers.json) at sizes
    the oracle finishes in seconds."""
    with open(os.path.join(GOLDEN, "known_answers.json")) as f:
        ka = json.load(f)
    g = bm.generate_random_bipartite(100_000, 100_000, 8.0, 1)
    k = ka["uniform/100000/8.0/1"]
    assert bm.csc_digest(g) == int(k["digest"]) and g.num_edges() == k["edges"] == 799_969
    r0, c0 = oracle.cheap_matching(g)
    assert int((r0 >= 0).sum()) == k["first_fit"] == 91_361
    st, r, c, ct = oracle.driver(g, r0, c0, tot=65536, kernel=1)
    assert int((r >= 0).sum()) == k["maximum"] == 99_961
    g = bm.generate_rmat(18, 16.0, 2024)
    k = ka["rmat/18/16/2024"]
    assert bm.csc_digest(g) == int(k["digest"]) and oracle.maximum(g) == k["maximum"]


def test_generator_restatement_matches(oracle):
    """oracle/gen_oracle.cpp (the reference arm's input builder, which must not
    load the product library) produces the same CSC as the product generators,
    and its uniform generator is the reference's generate_random_bipartite
    (csr_graph.cpp:92-112; digest of the 100K C1 graph from known_answers.json)."""
    from oracle import Generators
    gen = Generators(threads=4)
    pairs = [
        (gen.uniform(100_000, 100_000, 8.0, 1), bm.generate_random_bipartite(100_000, 100_000, 8.0, 1)),
        (gen.uniform(3_001, 2_000, 5.5, 77), bm.generate_random_bipartite(3_001, 2_000, 5.5, 77)),
        (gen.planted(200_000, 16.0, 2024), bm.generate_planted(200_000, 16.0, 2024)),
        (gen.rmat(14, 16.0, 2024), bm.generate_rmat(14, 16.0, 2024)),
        (gen.banded(300_000, 3, 0.05, 12345)[0], bm.generate_banded(300_000, 3, 0.05, 12345)[0]),
    ]
    for og, pg in pairs:
        assert (og.nc, og.nr) == (pg.nc, pg.nr)
        assert np.array_equal(og.cxadj, pg.cxadj), og.name
        assert np.array_equal(og.cadj, pg.cadj), og.name
    assert gen.banded(300_000, 3, 0.05, 12345)[1] == bm.generate_banded(300_000, 3, 0.05, 12345)[1]
    ka = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "known_answers.json")))
    g1 = pairs[0][0]
    assert str(bm.csc_digest(g1)) == ka["uniform/100000/8.0/1"]["digest"]
    r, c = gen.first_fit(g1)
    assert int((r >= 0).sum()) == ka["uniform/100000/8.0/1"]["first_fit"]
    r2, c2 = oracle.cheap_matching(g1)
    assert np.array_equal(r, r2) and np.array_equal(c, c2)
