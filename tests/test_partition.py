"""Multi-rank tests of the column-partitioned driver.

CPU (gloo, world 2 and 3): the host protocol of partition.py with the oracle's
restatement of the device backend. GPU (-m gpu): the bm_part_* kernels, two
ranks sharing cuda:0, records exchanged with gloo through host memory.
Checks: every rank ends with the same matching; it is valid, maximum, and its
cardinality equals the CPU oracle's maximum."""
import json
import os
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


def _run(world, backend, tmp_path, device_mode="gloo"):
    import torch.multiprocessing as mp
    import part_worker
    mp.spawn(part_worker.run, args=(world, _free_port(), backend, str(tmp_path), device_mode), nprocs=world, join=True)
    return [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]


def _check(results, oracle):
    gs = graphs()
    r0 = results[0]
    assert len(r0) == 3 * len(gs)
    for other in results[1:]:
        for a, b in zip(r0, other):  # replicas agree after the final broadcast
            assert a["card"] == b["card"] and a["rmatch"] == b["rmatch"] and a["cmatch"] == b["cmatch"]
    for rec in r0:
        g = gs[rec["graph"]]
        rm = np.array(rec["rmatch"], np.int32)
        cm = np.array(rec["cmatch"], np.int32)
        want = oracle.maximum(g)
        assert rec["card"] == want, (rec["graph"], rec["card"], want)
        assert int((rm >= 0).sum()) == want
        assert oracle.validate(g, rm, cm) == 0
        assert oracle.is_maximum(g, rm, cm) == 1


@pytest.mark.parametrize("world", [2, 3])
def test_partition_protocol_cpu_gloo(world, tmp_path, oracle):
    _check(_run(world, "cpu", tmp_path), oracle)


@pytest.mark.gpu
def test_partition_kernels_two_ranks_one_gpu(tmp_path, oracle):
    _check(_run(2, "gpu", tmp_path), oracle)


@pytest.mark.gpu
def test_partition_fused_p2p_exchange_two_ranks(tmp_path, oracle):
    """The fused exchange: records written by the expand kernel straight into
    both ranks' receive slabs (CUDA IPC), device-side arrival counting."""
    _check(_run(2, "gpu", tmp_path, device_mode="p2p"), oracle)


def test_column_range_and_slice():
    import paper_1303_1379_b200 as bm
    from paper_1303_1379_b200.partition import column_range, slice_csc
    g = bm.generate_random_bipartite(1001, 900, 3.0, 7)
    parts = [column_range(g.nc, r, 4) for r in range(4)]
    assert parts[0][0] == 0 and parts[-1][1] == g.nc
    assert all(parts[i][1] == parts[i + 1][0] for i in range(3))
    total = 0
    for lo, hi in parts:
        cx, adj = slice_csc(g, lo, hi)
        assert cx[0] == 0 and len(cx) == hi - lo + 1 and len(adj) == cx[-1]
        assert np.array_equal(adj, g.cadj[g.cxadj[lo]:g.cxadj[hi]])
        total += len(adj)
    assert total == g.num_edges()
