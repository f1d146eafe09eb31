"""Shared fixtures. `gpu`-marked tests need a B200 (run on the gpurun box);
everything else runs on CPU."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: large inputs (minutes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def engine():
    import paper_1303_1379_b200 as bm
    return bm.Engine(0)


def splitmix64(x: int) -> int:
    """kernel_grid.hpp:66-71 (used to size the acceptance corpus)."""
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def acceptance_corpus(count=1000):
    """The reference acceptance corpus (acceptance.cpp:78-108): `count` random
    graphs with nc, nr <= 200 and degrees {1,2,4,8}, then empty, edgeless,
    complete 12x9 and the fork graph."""
    import paper_1303_1379_b200 as bm
    degs = [1.0, 2.0, 4.0, 8.0]
    out = []
    for i in range(count):
        nc = 1 + splitmix64(2 * i) % 200
        nr = 1 + splitmix64(2 * i + 1) % 200
        g = bm.generate_random_bipartite(nc, nr, degs[i % 4], 10_000 + i)
        g.name = f"rand-{i}"
        out.append(g)
    out.append(bm.BipartiteCsr.from_edge_list(0, 0, [], "empty"))
    out.append(bm.BipartiteCsr.from_edge_list(7, 5, [], "edgeless"))
    out.append(bm.BipartiteCsr.from_edge_list(12, 9, [(c, r) for c in range(12) for r in range(9)], "complete"))
    out.append(fork_graph())
    return out


def fork_graph():
    """tests/oracles.hpp:59-61: c0 = {r0}, c1 = {r0, r1, r2}."""
    import paper_1303_1379_b200 as bm
    return bm.BipartiteCsr.from_edge_list(2, 3, [(0, 0), (1, 0), (1, 1), (1, 2)], "fork")


def fork_partial_matching():
    """test_gpu_match.cpp:30-35: only the shared row matched, c1-r0."""
    import paper_1303_1379_b200 as bm
    return bm.MatchingState(np.array([1, -1, -1], np.int32), np.array([-1, 0], np.int32))
