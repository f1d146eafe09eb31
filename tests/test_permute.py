"""permute_random (csr_graph.cpp:80-90, the paper's RCP experiments) on the
device: bm_permutation_pair must reproduce the reference's permutations, and
bm_permute_random must relabel the resident graph bit-identically to the
reference's permute_random (checked by CSC digest against oracle/_ref)."""
import numpy as np
import pytest

from oracle import Reference, have_reference

needs_ref = pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")


def host_permute(g, cp, rp):
    """Apply (cperm, rperm) on the host: the CSC of {(cp[c], rp[r])}, rows sorted."""
    import paper_1303_1379_b200 as bm
    cols = np.repeat(np.arange(g.nc, dtype=np.int64), np.diff(g.cxadj))
    return bm.BipartiteCsr.from_edge_list(g.nc, g.nr, list(zip(cp[cols].tolist(), rp[g.cadj].tolist())))


@needs_ref
@pytest.mark.parametrize("nc,nr,deg,seed,pseed", [(50, 40, 3.0, 1, 7), (3000, 2500, 4.0, 2, 99), (1, 1, 1.0, 3, 5)])
def test_permutation_pair_matches_reference(nc, nr, deg, seed, pseed):
    import paper_1303_1379_b200 as bm
    ref = Reference()
    g = bm.generate_random_bipartite(nc, nr, deg, seed)
    cp, rp = bm.permutation_pair(g.nc, g.nr, pseed)
    assert sorted(cp.tolist()) == list(range(g.nc)) and sorted(rp.tolist()) == list(range(g.nr))
    _, _, rcx, radj = ref.from_csc(g).permute(pseed).arrays()
    mine = host_permute(g, cp, rp)
    assert np.array_equal(mine.cxadj, rcx) and np.array_equal(mine.cadj, radj)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("nc,nr,deg,seed,pseed", [(3000, 2500, 4.0, 2, 99), (200000, 200000, 6.0, 4242, 3)])
def test_device_permute_matches_reference(engine, oracle, nc, nr, deg, seed, pseed):
    import paper_1303_1379_b200 as bm
    ref = Reference()
    g = bm.generate_random_bipartite(nc, nr, deg, seed)
    engine.upload(g, force=True)
    engine.permute_random(pseed)
    pg = engine.download_graph()
    _, _, rcx, radj = ref.from_csc(g).permute(pseed).arrays()
    assert np.array_equal(pg.cxadj, rcx) and np.array_equal(pg.cadj, radj)
    # the permuted graph matches to the same cardinality
    init = bm.cheap_matching(pg)
    engine.load_matching(init)
    card, ct, done = engine.run()
    assert done and card == oracle.maximum(g)


@pytest.mark.gpu
def test_device_permute_rmat_hubs(engine):
    import paper_1303_1379_b200 as bm
    g = bm.generate_rmat(14, 16.0, 5, permute=False)  # skewed: long columns go through the segmented sort
    engine.upload(g, force=True)
    engine.permute_random(11)
    pg = engine.download_graph()
    cp, rp = bm.permutation_pair(g.nc, g.nr, 11)
    mine = host_permute(g, cp, rp)
    assert np.array_equal(pg.cxadj, mine.cxadj) and np.array_equal(pg.cadj, mine.cadj)
