"""Parity of the sm_100a engine against the CPU oracle, through the C ABI.

The bar (north_star): the cardinality is bit-exact with the reference on the
same graph; the matched pairs may differ (race-resolved augmentation), so
every output is also checked to be a valid matching with no augmenting path
(validate + is_maximum, matching.cpp:70-131).
"""
import numpy as np
import pytest

import paper_1303_1379_b200 as bm
from conftest import acceptance_corpus, fork_graph, fork_partial_matching

pytestmark = pytest.mark.gpu

CONFIGS = [  # algorithms.cpp:19-27
    ("apfb-gpubfs", False, bm.BfsKernel.Gpubfs, False),
    ("apfb-wr", False, bm.BfsKernel.GpubfsWr, False),
    ("apsb-gpubfs", True, bm.BfsKernel.Gpubfs, False),
    ("apsb-wr", True, bm.BfsKernel.GpubfsWr, True),
]


def _check(oracle, g, res, want, init_card=None):
    m = res.matching
    assert oracle.validate(g, m.rmatch, m.cmatch) == 0, g.name
    assert bm.cardinality(m) == want, (g.name, bm.cardinality(m), want)
    assert oracle.is_maximum(g, m.rmatch, m.cmatch) == 1, g.name
    c = res.counters
    assert 1 <= c.outer_iterations <= g.nc + 1
    assert len(c.bfs_launches_per_iteration) == c.outer_iterations


@pytest.fixture(scope="module")
def corpus(oracle):
    graphs = acceptance_corpus(1000)
    return [(g, oracle.brute_force_maximum(g)) for g in graphs]


@pytest.mark.parametrize("cfg", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_corpus_given_init(engine, oracle, corpus, cfg):
    """acceptance.cpp:135-237 criterion 1 through the B200 engine (first-fit init)."""
    _, shortest, kernel, improved = cfg
    for g, want in corpus:
        init = bm.cheap_matching(g)
        res = engine.match(g, init, shortest=shortest, kernel=kernel, improved=improved)
        _check(oracle, g, res, want)


@pytest.mark.parametrize("init_mode", ["gpu_greedy", "gpu_ks"])
def test_corpus_gpu_init(engine, oracle, corpus, init_mode):
    for g, want in corpus[::3]:
        for _, shortest, kernel, improved in CONFIGS:
            res = engine.match(g, None, shortest=shortest, kernel=kernel, improved=improved, init_mode=init_mode)
            _check(oracle, g, res, want)
            # the GPU-built initial matching is maximal: no edge joins two free vertices
            assert res.counters.initial_cardinality <= want


def test_gpu_greedy_init_is_maximal(engine, oracle):
    g = bm.generate_random_bipartite(5000, 4000, 3.0, 77)
    res = engine.match(g, None, shortest=False, kernel=bm.BfsKernel.GpubfsWr, init_mode="gpu_greedy",
                       )
    assert res.counters.initial_cardinality > 0
    # from an empty init the result is still maximum
    _check(oracle, g, res, oracle.maximum(g))


def test_fork_graph_bfs_trace(engine):
    """test_gpu_match.cpp:51-71: GPUBFS on the fork graph, full expansion."""
    g = fork_graph()
    bfs, pred, rm, launches, found = engine.bfs_phase(g, fork_partial_matching(), kernel=bm.BfsKernel.Gpubfs)
    assert bfs.tolist() == [2, 3]
    assert pred.tolist() == [0, 1, 1]
    assert rm.tolist() == [1, -2, -2]
    assert launches == 2 and found


def test_fork_graph_improved_root_encoding(engine):
    """test_gpu_match.cpp:111-129: the root entry becomes -(endpoint row); the
    serial reference keeps r2 (-2); under races either endpoint is valid."""
    g = fork_graph()
    bfs, pred, rm, launches, found = engine.bfs_phase(g, fork_partial_matching(), shortest=True,
                                                      kernel=bm.BfsKernel.GpubfsWr, improved=True)
    assert bfs[0] in (-1, -2)
    assert bfs[1] == 3
    assert rm.tolist() == [1, -2, -2]
    assert found


def test_bfs_levels_match_queue_bfs(engine, oracle):
    """test_gpu_match.cpp:95-109: GPUBFS labels = queue-BFS depth + 2 (1 if unreachable)."""
    import conftest
    for i in range(60):
        nc = 1 + conftest.splitmix64(2 * i + 21) % 300
        nr = 1 + conftest.splitmix64(2 * i + 22) % 300
        g = bm.generate_random_bipartite(nc, nr, [1.0, 2.0, 4.0, 8.0][i % 4], 500 + i)
        init = bm.cheap_matching(g)
        depth = oracle.depths(g, init.rmatch, init.cmatch)
        bfs, *_ = engine.bfs_phase(g, init, kernel=bm.BfsKernel.Gpubfs)
        want = np.where(depth >= 0, depth + 2, 1)
        assert np.array_equal(bfs, want), i
    # and at a size where many CTAs race on every level
    g = bm.generate_random_bipartite(200000, 200000, 4.0, 3)
    init = bm.cheap_matching(g)
    depth = oracle.depths(g, init.rmatch, init.cmatch)
    bfs, *_ = engine.bfs_phase(g, init, kernel=bm.BfsKernel.Gpubfs)
    assert np.array_equal(bfs, np.where(depth >= 0, depth + 2, 1))


def test_edge_cases(engine, oracle):
    empty = bm.BipartiteCsr.from_edge_list(0, 0, [])
    r = engine.match(empty, bm.MatchingState.unmatched(0, 0))
    assert r.counters.outer_iterations == 1 and r.counters.bfs_launches_per_iteration == [1]
    edgeless = bm.BipartiteCsr.from_edge_list(3, 4, [])
    init = bm.MatchingState.unmatched(3, 4)
    r = engine.match(edgeless, init)  # test_gpu_match.cpp:283-291
    assert np.array_equal(r.matching.rmatch, init.rmatch) and r.counters.outer_iterations == 1
    one = bm.BipartiteCsr.from_edge_list(1, 1, [(0, 0)])
    r = engine.match(one, bm.MatchingState.unmatched(1, 1))
    assert r.matching.rmatch.tolist() == [0] and r.matching.cmatch.tolist() == [0]
    comp = bm.BipartiteCsr.from_edge_list(3, 3, [(c, rr) for c in range(3) for rr in range(3)])
    r = engine.match(comp, bm.cheap_matching(comp), shortest=True, kernel=bm.BfsKernel.Gpubfs)
    assert r.counters.outer_iterations == 1 and r.counters.bfs_launches_per_iteration == [1]
    fork = fork_graph()
    r = engine.match(fork, bm.cheap_matching(fork), kernel=bm.BfsKernel.Gpubfs)  # test_gpu_match.cpp:274-281
    assert bm.cardinality(r.matching) == 2 and r.counters.outer_iterations == 1
    r = engine.match(fork, fork_partial_matching(), shortest=True, kernel=bm.BfsKernel.GpubfsWr, improved=True)
    assert bm.cardinality(r.matching) == 2 and oracle.is_maximum(fork, r.matching.rmatch, r.matching.cmatch) == 1


def test_observer_phase_invariants(engine, oracle):
    """test_gpu_match.cpp:357-377: every phase leaves a valid matching and a
    monotone cardinality; the per-phase events match the counters."""
    g = bm.generate_random_bipartite(20000, 20000, 3.0, 11)
    for _, shortest, kernel, improved in CONFIGS:
        events = []

        def obs(ev):
            assert oracle.validate(g, ev.state.rmatch, ev.state.cmatch) == 0
            assert ev.cardinality_after >= ev.cardinality_before
            assert bm.cardinality(ev.state) == ev.cardinality_after
            events.append(ev)

        res = engine.match(g, bm.cheap_matching(g), shortest=shortest, kernel=kernel, improved=improved,
                           observer=obs)
        assert len(events) == res.counters.outer_iterations
        assert [e.bfs_launches for e in events] == res.counters.bfs_launches_per_iteration
        assert not events[-1].augmenting_path_found
        assert all(e.augmenting_path_found for e in events[:-1])


def test_observer_exception_propagates(engine):
    g = bm.generate_random_bipartite(1000, 1000, 2.0, 5)

    def boom(ev):
        raise KeyError("stop")

    with pytest.raises(KeyError):
        engine.match(g, bm.cheap_matching(g), observer=boom)


def test_errors(engine):
    g = fork_graph()
    with pytest.raises(bm.LogicError):  # gpu_match.cpp:272-274
        engine.match(g, bm.cheap_matching(g), kernel=bm.BfsKernel.Gpubfs, improved=True)
    bad = bm.MatchingState(np.array([0, 0, -1], np.int32), np.array([0, -1], np.int32))  # asymmetric
    with pytest.raises(ValueError):
        engine.match(g, bad)
    pending = bm.MatchingState(np.array([-2, -1, -1], np.int32), np.array([-1, -1], np.int32))
    with pytest.raises(ValueError):
        engine.match(g, pending)
    broken = bm.BipartiteCsr(2, 3, np.array([0, 1, 4], np.int64), np.array([0, 0, 1, 5], np.int32))
    with pytest.raises(ValueError):
        engine.upload(broken)
    nonmono = bm.BipartiteCsr(2, 3, np.array([0, 3, 2], np.int64), np.array([0, 1], np.int32))
    with pytest.raises(ValueError):
        engine.upload(nonmono)
    # the engine stays usable after errors
    r = engine.match(g, bm.cheap_matching(g))
    assert bm.cardinality(r.matching) == 2


def test_resident_run_and_resume(engine, oracle):
    g = bm.generate_random_bipartite(100000, 100000, 8.0, 1)
    init = bm.cheap_matching(g)
    engine.upload(g)
    engine.load_matching(init)
    cards = []
    for _ in range(3):
        card, ct, done = engine.run(kernel=bm.BfsKernel.GpubfsWr)
        assert done
        cards.append(card)
    assert cards == [99961] * 3  # reference known answer
    m = engine.download()
    assert oracle.validate(g, m.rmatch, m.cmatch) == 0
    # stop after one phase, then resume to the maximum
    card1, ct1, done1 = engine.run(kernel=bm.BfsKernel.GpubfsWr, max_phases=1)
    assert not done1 and card1 > bm.cardinality(init)
    card2, ct2, done2 = engine.run(kernel=bm.BfsKernel.GpubfsWr, resume=True)
    assert done2 and card2 == 99961
    assert ct2.outer_iterations >= 2


@pytest.mark.parametrize("nc,deg,seed,want", [
    (100000, 8.0, 1, 99961),     # C1; SURVEY §8c known answers produced by the reference
    (200000, 6.0, 4242, 199472),  # acceptance criterion 7 instance
    (1000000, 8.0, 1, 999679),
])
def test_reference_known_answers(engine, oracle, nc, deg, seed, want):
    g = bm.generate_random_bipartite(nc, nc, deg, seed)
    init = bm.cheap_matching(g)
    for _, shortest, kernel, improved in CONFIGS:
        res = engine.match(g, init, shortest=shortest, kernel=kernel, improved=improved)
        _check(oracle, g, res, want)


def test_planted_and_banded(engine, oracle):
    g = bm.generate_planted(1_000_000, 16.0, 2024)
    res = engine.match(g, bm.cheap_matching(g))
    _check(oracle, g, res, 1_000_000)
    res = engine.match(g, bm.cheap_matching(g), shortest=True, kernel=bm.BfsKernel.GpubfsWr, improved=True)
    _check(oracle, g, res, 1_000_000)
    gb, live = bm.generate_banded(1_000_000, 3, 0.05, 12345)
    res = engine.match(gb, bm.cheap_matching(gb))
    _check(oracle, gb, res, live)


def test_rmat_skewed(engine, oracle):
    g = bm.generate_rmat(18, 16.0, 2024)
    want = oracle.maximum(g)
    init = bm.cheap_matching(g)
    for _, shortest, kernel, improved in CONFIGS:
        res = engine.match(g, init, shortest=shortest, kernel=kernel, improved=improved)
        _check(oracle, g, res, want)


def test_verify_matches_oracle(engine, oracle):
    g = bm.generate_random_bipartite(50000, 40000, 3.0, 8)
    init = bm.cheap_matching(g)
    v, ismax, card = engine.verify(g, init)
    assert v == 0 and card == bm.cardinality(init)
    assert ismax == (oracle.is_maximum(g, init.rmatch, init.cmatch) == 1)
    res = engine.match(g, init)
    v, ismax, card = engine.verify(g, res.matching)
    assert v == 0 and ismax and card == oracle.maximum(g)
    bad = res.matching.copy()
    r = int(np.flatnonzero(bad.rmatch >= 0)[0])
    bad.rmatch[r] = -2
    v, _, _ = engine.verify(g, bad)
    assert v == oracle.validate(g, bad.rmatch, bad.cmatch) > 0


def test_unsorted_columns_and_upload_checks(engine, oracle):
    """check_csr semantics at upload (csr_graph.cpp:45-64): rows out of range are
    rejected; unsorted columns are accepted (the kernels do not rely on order) and
    the verifier falls back to a linear scan."""
    g = bm.generate_random_bipartite(20000, 15000, 5.0, 77)
    rng = np.random.default_rng(5)
    adj = g.cadj.copy()
    for c in range(0, g.nc, 3):  # reverse every third column
        a, b = g.cxadj[c], g.cxadj[c + 1]
        adj[a:b] = adj[a:b][::-1]
    ug = bm.BipartiteCsr(g.nc, g.nr, g.cxadj.copy(), adj)
    init = bm.cheap_matching(ug)
    res = engine.match(ug, init)
    want = oracle.maximum(g)
    assert bm.cardinality(res.matching) == want
    viol, ismax, card = engine.verify(ug, res.matching)
    assert viol == 0 and ismax and card == want
    bad = g.cadj.copy()
    bad[int(rng.integers(0, len(bad)))] = g.nr  # one row id out of range
    with pytest.raises(ValueError):
        engine.upload(bm.BipartiteCsr(g.nc, g.nr, g.cxadj.copy(), bad), force=True)
    engine.upload(g, force=True)
    res = engine.match(g, bm.cheap_matching(g))
    assert bm.cardinality(res.matching) == want


@pytest.mark.parametrize("left", ["1", "0"], ids=["leftover_lists", "screen_all"])
def test_bottom_up_levels_parity(oracle, corpus, monkeypatch, left):
    """Every level bottom-up (BM_BU_FRAC=0, no single-CTA levels): the pulled
    levels must give the same maxima as the oracle on the corpus and on larger
    graphs, under every driver/kernel combination — with consecutive pulled
    levels taking their candidates from the level before's leftover list, and
    with every level screening every row (BM_BU_LEFT=0)."""
    monkeypatch.setenv("BM_BU_FRAC", "0")
    monkeypatch.setenv("BM_SOLO_EDGES", "0")
    monkeypatch.setenv("BM_BU_LEFT", left)
    eng = bm.Engine(0)
    eng.bottom_up = True
    graphs = [g for g, _ in corpus[:120] + corpus[-4:]] + [
        bm.generate_random_bipartite(20000, 20000, 4.0, 3), bm.generate_planted(30000, 8.0, 4), bm.generate_rmat(13, 8.0, 2)]
    for g in graphs:
        init = bm.cheap_matching(g)
        want = oracle.maximum(g)
        for shortest, kernel, improved in [(False, bm.BfsKernel.GpubfsWr, False), (True, bm.BfsKernel.GpubfsWr, True),
                                           (False, bm.BfsKernel.Gpubfs, False), (True, bm.BfsKernel.Gpubfs, False)]:
            res = eng.match(g, init, shortest=shortest, kernel=kernel, improved=improved)
            m = res.matching
            assert bm.cardinality(m) == want, (g.name, shortest, kernel)
            assert oracle.validate(g, m.rmatch, m.cmatch) == 0
            assert oracle.is_maximum(g, m.rmatch, m.cmatch) == 1
    eng.close()


def test_bottom_up_auto_decision_and_row_index(oracle, monkeypatch):
    """BM_BU_AUTO: small graphs push; a large, even-degree graph pulls its dense
    levels. The row index the pulled levels read is built by the bucketed
    two-pass transpose; forcing AUTO on for small graphs (so the index is
    built for graphs of every shape, including empty columns and rows) must
    keep every maximum."""
    eng = bm.Engine(0)
    small = bm.generate_random_bipartite(20000, 20000, 8.0, 1)
    eng.upload(small)
    assert not eng.bottom_up_auto()
    big = bm.generate_random_bipartite(1 << 21, 1 << 21, 9.0, 2)
    eng.upload(big, force=True)
    assert eng.bottom_up_auto() == 1  # qualifies; pulls once the row index is prepared
    eng.prepare_row_index()
    init = bm.cheap_matching(big)
    res = eng.match(big, init)  # default "auto": pulled levels
    eng.bottom_up = False
    push = eng.match(big, init)
    assert bm.cardinality(res.matching) == bm.cardinality(push.matching)
    viol, ismax, _ = eng.verify(big, res.matching)
    assert viol == 0 and ismax
    eng.bottom_up = "auto"
    monkeypatch.setenv("BM_BU_AUTO", "1")
    monkeypatch.setenv("BM_BU_FRAC", "0")
    monkeypatch.setenv("BM_SOLO_EDGES", "0")
    for g in [small, bm.generate_rmat(14, 8.0, 5), bm.generate_banded(30000, 3, 0.1, 6)[0],
              bm.BipartiteCsr.from_edge_list(5, 4, [(1, 0), (1, 3), (4, 3)])]:
        eng.upload(g, force=True)
        assert eng.bottom_up_auto() == 2
        m = eng.match(g, bm.cheap_matching(g)).matching
        assert bm.cardinality(m) == oracle.maximum(g)
        assert oracle.validate(g, m.rmatch, m.cmatch) == 0
    eng.close()


def test_mixed_pushed_and_pulled_levels_parity(oracle, corpus, monkeypatch):
    """AUTO forced on (BM_BU_AUTO=1) with the default pull threshold: levels
    switch between pushed and pulled as the frontier grows and shrinks, and
    every driver/kernel combination must still reach the oracle's maximum."""
    monkeypatch.setenv("BM_BU_AUTO", "1")
    eng = bm.Engine(0)
    graphs = [g for g, _ in corpus[::5]] + [bm.generate_random_bipartite(30000, 30000, 8.0, 7),
                                             bm.generate_planted(40000, 12.0, 8)]
    for g in graphs:
        eng.upload(g, force=True)
        init = bm.cheap_matching(g)
        want = oracle.maximum(g)
        for shortest, kernel, improved in [(False, bm.BfsKernel.GpubfsWr, False), (True, bm.BfsKernel.GpubfsWr, True),
                                           (False, bm.BfsKernel.Gpubfs, False)]:
            m = eng.match(g, init, shortest=shortest, kernel=kernel, improved=improved).matching
            assert bm.cardinality(m) == want, (g.name, shortest, kernel)
            assert oracle.validate(g, m.rmatch, m.cmatch) == 0
    eng.close()


@pytest.mark.parametrize("bounds", [{}, {"BM_LATE_BCAP": "40", "BM_LATE_FCAP": "200", "BM_LATE_BLV": "2"},
                                    {"BM_LATE_ROOTS": "2000000000"}], ids=["default", "tight", "every_phase"])
def test_late_phase_parity(oracle, corpus, monkeypatch, bounds):
    """Late phases (BM_LATE=1; bm_kernels.cuh late_phase): phases with few roots
    first try a bounded meet-in-the-middle search whose vertex-disjoint paths
    are flipped without FIX; a late phase that finds nothing hands over to a
    full phase, which alone ends the driver. Every maximum must equal the
    oracle's, the matching must be valid and maximum, and each late phase must
    augment (strictly increasing cardinality per recorded phase). A late phase
    that finds nothing but whose backward search from every free row ran to its
    end without meeting a free column ends the run (no augmenting path exists);
    the oracle's is_maximum checks those endings too. All this with the
    default bounds, with bounds so tight that most late phases give up, and
    with every phase tried late (from the unmatched state too)."""
    monkeypatch.setenv("BM_LATE", "1")
    for k, v in bounds.items():
        monkeypatch.setenv(k, v)
    eng = bm.Engine(0)
    eng.bottom_up = True
    graphs = [g for g, _ in corpus[::4]] + [
        bm.generate_random_bipartite(20000, 20000, 4.0, 3), bm.generate_random_bipartite(30000, 20000, 3.0, 5),
        bm.generate_random_bipartite(20000, 30000, 3.0, 6), bm.generate_planted(30000, 8.0, 4),
        bm.generate_rmat(13, 8.0, 2), bm.generate_banded(30000, 3, 0.1, 6)[0]]
    late_paths = proofs = 0
    for g in graphs:
        want = oracle.maximum(g)
        for init in [bm.cheap_matching(g), None]:
            events = []
            res = eng.match(g, init, kernel=bm.BfsKernel.GpubfsWr, observer=events.append)
            m = res.matching
            assert bm.cardinality(m) == want, g.name
            assert oracle.validate(g, m.rmatch, m.cmatch) == 0
            assert oracle.is_maximum(g, m.rmatch, m.cmatch) == 1
            for ev in events[:-1]:
                assert ev.cardinality_after > ev.cardinality_before, g.name
            st = eng.debug_stats()
            late_paths += st["late_paths"]
            proofs += st["late_proofs"]
    assert late_paths > 0
    if not bounds:
        assert proofs > 0  # some runs end on a late phase's exhausted backward search
    eng.close()


# ---- failure paths of run_driver (fault injection through bm_debug_set) ----

@pytest.mark.parametrize("cfg", CONFIGS, ids=[c[0] for c in CONFIGS])
@pytest.mark.parametrize("bottom_up", [False, True])
def test_serial_retry_after_no_progress_phase(oracle, cfg, bottom_up, monkeypatch):
    """A raced phase that found paths but augmented none is rerun with a serial
    ALTERNATE (gpu_match.cpp:328-343): phase 1's parallel ALTERNATE is made a
    no-op, so the device must take the retry, count it, and still reach the
    maximum."""
    if bottom_up:
        monkeypatch.setenv("BM_BU_FRAC", "0")  # every wide level pulled
    _, shortest, kernel, improved = cfg
    eng = bm.Engine(0)
    g = bm.generate_random_bipartite(20000, 20000, 6.0, 3)
    init = bm.cheap_matching(g)
    want = oracle.maximum(g)
    eng.debug_set(bm.Engine.DEBUG_SKIP_ALTERNATE_PHASE, 1)
    eng.upload(g)
    eng.load_matching(init)
    card, ct, done = eng.run(shortest=shortest, kernel=kernel, improved=improved, bottom_up=bottom_up)
    assert done and card == want
    assert ct.serial_retries == 1
    m = eng.download()
    assert oracle.validate(g, m.rmatch, m.cmatch) == 0 and oracle.is_maximum(g, m.rmatch, m.cmatch) == 1
    # the retried phase is one outer iteration (its launches include both BFS passes)
    res = eng.match(g, init, shortest=shortest, kernel=kernel, improved=improved)
    _check(oracle, g, res, want)
    assert res.counters.serial_retries == 1
    events = []
    eng.match(g, init, shortest=shortest, kernel=kernel, improved=improved, observer=events.append)
    assert events[0].serial_retry and events[0].cardinality_after > events[0].cardinality_before
    assert not any(e.serial_retry for e in events[1:])
    eng.debug_set(bm.Engine.DEBUG_SKIP_ALTERNATE_PHASE, 0)
    res = eng.match(g, init, shortest=shortest, kernel=kernel, improved=improved)
    assert res.counters.serial_retries == 0


def test_phase_bound_exceeded_raises(engine, oracle):
    """More than the bound's phases -> runtime_error (gpu_match.cpp:313-320),
    BM_ERR_BOUND_EXCEEDED at the C ABI; the handle stays usable."""
    g = bm.generate_random_bipartite(50000, 50000, 6.0, 9)
    init = bm.cheap_matching(g)
    want = oracle.maximum(g)
    res = engine.match(g, init)
    assert res.counters.outer_iterations >= 3
    engine.debug_set(bm.Engine.DEBUG_PHASE_BOUND, 2)
    try:
        with pytest.raises(RuntimeError, match="bound"):
            engine.match(g, init)
        engine.upload(g)
        engine.load_matching(init)
        with pytest.raises(RuntimeError, match="bound"):
            engine.run()
        # a bound the run fits under is not an error
        engine.debug_set(bm.Engine.DEBUG_PHASE_BOUND, res.counters.outer_iterations + 8)
        _check(oracle, g, engine.match(g, init), want)
    finally:
        engine.debug_set(bm.Engine.DEBUG_PHASE_BOUND, 0)
    _check(oracle, g, engine.match(g, init), want)


def test_initial_matching_pair_must_be_an_edge(engine):
    """validate (matching.cpp:70-104): a matched (row, col) pair that is not an
    edge makes the initial matching invalid — including a column with no edges
    at all — on both the host-init path (bm_match) and the resident path."""
    # c0 = {r0}, c1 = {} (degree 0), c2 = {r1, r2}
    g = bm.BipartiteCsr(3, 3, np.array([0, 1, 1, 3], np.int64), np.array([0, 1, 2], np.int32))
    cases = [
        bm.MatchingState(np.array([1, -1, -1], np.int32), np.array([-1, 0, -1], np.int32)),  # c1-r0, deg(c1)=0
        bm.MatchingState(np.array([-1, -1, -1], np.int32), np.array([-1, -1, -1], np.int32)),
        bm.MatchingState(np.array([2, -1, -1], np.int32), np.array([-1, -1, 0], np.int32)),  # c2-r0 not an edge
    ]
    for i, m in enumerate(cases):
        if i == 1:
            assert bm.cardinality(engine.match(g, m).matching) == 2
            continue
        with pytest.raises(ValueError):
            engine.match(g, m)
        engine.upload(g, force=True)
        engine.load_matching(m)
        with pytest.raises(ValueError):
            engine.run()
    gu = bm.BipartiteCsr(2, 3, np.array([0, 2, 4], np.int64), np.array([2, 0, 1, 2], np.int32))  # unsorted c0
    ok = bm.MatchingState(np.array([0, -1, -1], np.int32), np.array([0, -1], np.int32))
    assert bm.cardinality(engine.match(gu, ok).matching) == 2
    bad = bm.MatchingState(np.array([-1, 0, -1], np.int32), np.array([1, -1], np.int32))  # c0-r1 not an edge
    with pytest.raises(ValueError):
        engine.match(gu, bad)
    r = engine.match(g, bm.cheap_matching(g))  # still usable
    assert bm.cardinality(r.matching) == 2


def test_asymmetric_initial_matching_rejected(engine, oracle):
    """The setup's row check is a count (matched rows == matched columns whose
    row points back), not a gather: a row that claims a column which does not
    point back must still be caught, on the in-kernel (bm_match) and the
    load-time (bm_load_matching) checks, while valid matchings pass."""
    g = bm.generate_random_bipartite(3000, 3000, 4.0, 5)
    good = bm.cheap_matching(g)
    assert bm.cardinality(engine.match(g, good).matching) == oracle.maximum(g)
    c0 = int(np.flatnonzero(good.cmatch >= 0)[0])
    r0 = int(good.cmatch[c0])
    free_rows = np.flatnonzero(good.rmatch < 0)
    bad1 = good.copy()
    bad1.rmatch[free_rows[0]] = c0  # a second row claims c0, which points to r0
    bad2 = good.copy()
    bad2.cmatch[c0] = -1  # r0 still claims c0, which now points nowhere
    bad3 = good.copy()
    bad3.rmatch[r0] = -1  # c0 claims r0, which points nowhere
    for m in (bad1, bad2, bad3):
        with pytest.raises(ValueError):
            engine.match(g, m)
        engine.upload(g, force=True)
        engine.load_matching(m)
        with pytest.raises(ValueError):
            engine.run()
    assert bm.cardinality(engine.match(g, good).matching) == oracle.maximum(g)


@pytest.mark.parametrize("spec", [{}, {"BM_BU_FRAC": "1.0"}, {"BM_BU_ALPHA": "100", "BM_SOLO_EDGES": "0"}])
def test_lazy_frontier_self_check(oracle, monkeypatch, spec):
    """Pulled-capable runs hand wide levels on as (col, root) pairs and build
    edge-tiled entries only for levels that are pushed (materialize). BM_CHECK=1
    makes the kernel verify every pushed level's entries and granule index
    before expanding it (a failed check is a CudaError). Skewed graph, repeated
    runs: the check once caught a race between a level's count and the next
    level's reservations."""
    monkeypatch.setenv("BM_CHECK", "1")
    for k, v in spec.items():
        monkeypatch.setenv(k, v)
    g = bm.generate_rmat(20, 16.0, 7)
    want = oracle.maximum(g)
    init = bm.cheap_matching(g)
    eng = bm.Engine(0)
    eng.upload(g)
    eng.load_matching(init)
    eng.prepare_row_index()
    for _ in range(4):
        for _, shortest, kernel, improved in CONFIGS:
            card, ct, done = eng.run(shortest=shortest, kernel=kernel, improved=improved, bottom_up=True)
            assert done and card == want
    m = eng.download()
    assert oracle.validate(g, m.rmatch, m.cmatch) == 0 and oracle.is_maximum(g, m.rmatch, m.cmatch) == 1


@pytest.mark.parametrize("spec", [{}, {"BM_PB_SLACK": "0", "BM_PB_MAX": "20000"}], ids=["regions", "overflow"])
def test_bucketed_push_parity(oracle, corpus, monkeypatch, spec):
    """Bucketed pushed levels (push_bucketed): forced on every pushed level of
    pulling runs (interleaved row state, no single-CTA levels, nothing pulled);
    with no slack in the bucket regions the skewed graphs also take the overflow
    region. Same maxima as the oracle under every driver/kernel combination."""
    env = {"BM_ROW_LAYOUT": "interleave", "BM_PB_MIN": "0", "BM_SOLO_EDGES": "0", "BM_BU_AUTO": "1",
           "BM_BU_FRAC": "2.0"}
    env.update(spec)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    eng = bm.Engine(0)
    eng.bottom_up = True
    graphs = [g for g, _ in corpus[:200:4] + corpus[-4:]] + [
        bm.generate_random_bipartite(20000, 20000, 4.0, 3), bm.generate_planted(30000, 8.0, 4),
        bm.generate_rmat(13, 8.0, 2), bm.generate_banded(20000, 3, 0.1, 7)[0]]
    for g in graphs:
        init = bm.cheap_matching(g)
        want = oracle.maximum(g)
        for shortest, kernel, improved in [(False, bm.BfsKernel.GpubfsWr, False), (True, bm.BfsKernel.GpubfsWr, True),
                                           (False, bm.BfsKernel.Gpubfs, False), (True, bm.BfsKernel.Gpubfs, False)]:
            res = eng.match(g, init, shortest=shortest, kernel=kernel, improved=improved)
            m = res.matching
            assert bm.cardinality(m) == want, (g.name, shortest, kernel)
            assert oracle.validate(g, m.rmatch, m.cmatch) == 0
            assert oracle.is_maximum(g, m.rmatch, m.cmatch) == 1
    tl = [k for k, _, _ in eng.timeline()]
    assert "bucketed" in tl  # the path ran (last run's timeline)
    eng.close()


def test_last_phase_launches_match_counters(engine, oracle):
    """bm_last_phase_launches returns the per-phase BFS launch counts that
    bm_match reports in PhaseCounters (the C++ shim fetches long runs this way)."""
    g = bm.generate_random_bipartite(50000, 50000, 6.0, 21)
    res = engine.match(g, bm.cheap_matching(g))
    launches = engine.last_phase_launches()
    assert launches == list(res.counters.bfs_launches_per_iteration)
    assert len(launches) == res.counters.outer_iterations >= 1


@pytest.mark.parametrize("spec", [{}, {"BM_PB_SLACK": "0"}], ids=["regions", "overflow"])
def test_bucketed_prep_parity(oracle, corpus, monkeypatch, spec):
    """Bucketed bu_prep (column buckets, bu_prep_bucketed): forced on every pulled
    level with roots (interleaved row state, every level pulled); with no slack
    in the bucket regions the skewed graphs take the overflow region. Same maxima
    as the oracle under every driver/kernel combination."""
    env = {"BM_ROW_LAYOUT": "interleave", "BM_PP_MIN": "0", "BM_SOLO_EDGES": "0", "BM_BU_AUTO": "1",
           "BM_BU_FRAC": "0"}
    env.update(spec)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    eng = bm.Engine(0)
    eng.bottom_up = True
    graphs = [g for g, _ in corpus[:200:4] + corpus[-4:]] + [
        bm.generate_random_bipartite(20000, 20000, 4.0, 3), bm.generate_planted(30000, 8.0, 4),
        bm.generate_rmat(13, 8.0, 2), bm.generate_banded(20000, 3, 0.1, 7)[0]]
    for g in graphs:
        init = bm.cheap_matching(g)
        want = oracle.maximum(g)
        for shortest, kernel, improved in [(False, bm.BfsKernel.GpubfsWr, False), (True, bm.BfsKernel.GpubfsWr, True),
                                           (False, bm.BfsKernel.Gpubfs, False)]:
            m = eng.match(g, init, shortest=shortest, kernel=kernel, improved=improved).matching
            assert bm.cardinality(m) == want, (g.name, shortest, kernel)
            assert oracle.validate(g, m.rmatch, m.cmatch) == 0
            assert oracle.is_maximum(g, m.rmatch, m.cmatch) == 1
    eng.close()
