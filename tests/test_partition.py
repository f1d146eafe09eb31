"""Multi-rank tests of the multi-GPU engine.

CPU (gloo, world 2 and 3): the host protocol of partition.py — slicing,
peer-blob exchange, row-index barrier, load/launch ordering, gathering the
slices — with the CPU stand-in for the device (oracle.partition_ref).
GPU (-m gpu): the real multi-GPU kernels, a team of 2-4 ranks in one process
sharing cuda:0 (one stream and one cooperative launch per rank; every rank
reaches the others' state through peer pointers, as over NVLink).
Checks: every rank ends with the same matching; it is valid, maximum, and its
cardinality equals the CPU oracle's maximum."""
import json
import socket

import numpy as np
import pytest

from part_worker import graphs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, tmp_path):
    import torch.multiprocessing as mp
    import part_worker
    mp.spawn(part_worker.run, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    return [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]


def _check_one(g, card, rm, cm, oracle):
    want = oracle.maximum(g)
    assert card == want, (g.name, card, want)
    assert int((rm >= 0).sum()) == want
    assert oracle.validate(g, rm, cm) == 0
    assert oracle.is_maximum(g, rm, cm) == 1


@pytest.mark.parametrize("world", [2, 3])
def test_partition_protocol_cpu_gloo(world, tmp_path, oracle):
    results = _run(world, tmp_path)
    gs = graphs()
    r0 = results[0]
    assert len(r0) == 3 * len(gs)
    for other in results[1:]:  # every rank gathered the same matching
        for a, b in zip(r0, other):
            assert a["card"] == b["card"] and a["rmatch"] == b["rmatch"] and a["cmatch"] == b["cmatch"]
    for rec in r0:
        _check_one(gs[rec["graph"]], rec["card"], np.array(rec["rmatch"], np.int32),
                   np.array(rec["cmatch"], np.int32), oracle)


def test_partition_bounds_and_slices():
    import paper_1303_1379_b200 as bm
    from paper_1303_1379_b200.partition import column_range, partition_bounds, slice_csc
    g = bm.generate_random_bipartite(1001, 900, 3.0, 7)
    for world in (1, 2, 3, 4, 8):
        b = partition_bounds(g.nc, world)
        assert b[0] == 0 and b[-1] == g.nc and all(b[i] <= b[i + 1] for i in range(world))
        assert all(x % 32 == 0 for x in b[1:-1])  # bitmap words never straddle two ranks
        total = 0
        for q in range(world):
            lo, hi = column_range(g.nc, q, world)
            assert (lo, hi) == (b[q], b[q + 1])
            cx, adj = slice_csc(g, lo, hi)
            assert cx[0] == 0 and len(cx) == hi - lo + 1 and len(adj) == cx[-1]
            assert np.array_equal(adj, g.cadj[g.cxadj[lo]:g.cxadj[hi]])
            total += len(adj)
        assert total == g.num_edges()
    assert partition_bounds(10, 4) == [0, 10, 10, 10, 10]  # ranks may own nothing


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_multigpu_team_one_device(world, oracle):
    import paper_1303_1379_b200 as bm
    from paper_1303_1379_b200.partition import LocalTeam
    team = LocalTeam(world)
    gs = graphs() + [bm.generate_random_bipartite(200000, 200000, 6.0, 4242)]
    for gi, g in enumerate(gs):
        init = bm.cheap_matching(g)
        pulled = gi % 2 == 1
        team.upload(g, row_index=pulled)
        for shortest, kernel, improved in [(False, bm.BfsKernel.GpubfsWr, False), (True, bm.BfsKernel.GpubfsWr, True),
                                           (False, bm.BfsKernel.Gpubfs, False)]:
            res, m = team.match(init, shortest=shortest, kernel=kernel, improved=improved,
                                bottom_up="on" if pulled else "off")
            assert bm.cardinality(m) == res.cardinality
            _check_one(g, res.cardinality, m.rmatch, m.cmatch, oracle)
    team.close()


@pytest.mark.gpu
def test_multigpu_pulled_levels_every_level(oracle, monkeypatch):
    """Every level pulled (BM_BU_FRAC=0) across a team of 3: the frontier
    bitmap replicas, the distributed row index and the routed winners."""
    import paper_1303_1379_b200 as bm
    from paper_1303_1379_b200.partition import LocalTeam
    monkeypatch.setenv("BM_BU_FRAC", "0")
    team = LocalTeam(3)
    for g in [bm.generate_random_bipartite(20000, 20000, 4.0, 3), bm.generate_planted(30000, 8.0, 4),
              bm.generate_rmat(13, 8.0, 2)]:
        init = bm.cheap_matching(g)
        team.upload(g, row_index=True)
        for shortest, kernel, improved in [(False, bm.BfsKernel.GpubfsWr, False), (True, bm.BfsKernel.GpubfsWr, True)]:
            res, m = team.match(init, shortest=shortest, kernel=kernel, improved=improved, bottom_up="on")
            _check_one(g, res.cardinality, m.rmatch, m.cmatch, oracle)
    team.close()


@pytest.mark.gpu
def test_multigpu_upload_checks_and_reuse(oracle):
    """The slice is checked on the device (check_csr, csr_graph.cpp:45-64): a row
    out of range or decreasing offsets fail the upload with invalid_argument;
    re-uploading graphs of other sizes into the same team (buffers grown, not
    reallocated, when they fit) keeps every maximum."""
    import numpy as np
    import paper_1303_1379_b200 as bm
    from paper_1303_1379_b200.partition import LocalTeam
    team = LocalTeam(2)
    g = bm.generate_random_bipartite(20000, 15000, 5.0, 77)
    bad = g.cadj.copy()
    bad[len(bad) // 3] = g.nr
    with pytest.raises(ValueError):
        team.upload(bm.BipartiteCsr(g.nc, g.nr, g.cxadj.copy(), bad))
    cx = g.cxadj.copy()
    cx[g.nc // 4] = cx[g.nc // 4 + 1] + 2
    with pytest.raises(ValueError):
        team.upload(bm.BipartiteCsr(g.nc, g.nr, cx, g.cadj.copy()))
    for h in [g, bm.generate_random_bipartite(5000, 6000, 3.0, 5), bm.generate_rmat(14, 8.0, 9), g]:
        team.upload(h, row_index=True)
        res, m = team.match(bm.cheap_matching(h), bottom_up="auto")
        _check_one(h, res.cardinality, m.rmatch, m.cmatch, oracle)
    team.close()
