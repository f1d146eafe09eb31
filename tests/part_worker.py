"""Worker for the multi-rank tests of the multi-GPU protocol (spawned with
torch.multiprocessing over gloo). Each rank builds the same graphs, runs the
partitioned driver (partition.PartitionedMatcher) with the CPU stand-in for
the device (oracle.partition_ref.CpuRank) and saves the gathered matching."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def graphs():
    import paper_1303_1379_b200 as bm
    from conftest import acceptance_corpus
    gs = acceptance_corpus(24)  # small random corpus + empty, edgeless, complete, fork
    gs.append(bm.generate_random_bipartite(3000, 2500, 3.0, 41))
    gs.append(bm.generate_planted(2000, 4.0, 5))
    g, _ = bm.generate_banded(3000, 3, 0.05, 9)
    gs.append(g)
    gs.append(bm.generate_rmat(11, 8.0, 3))
    return gs


def run(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1303_1379_b200 as bm
    from oracle.partition_ref import CpuRank
    from paper_1303_1379_b200.partition import DistTransport, PartitionedMatcher
    x = DistTransport()
    pm = PartitionedMatcher(CpuRank(rank, world, x), x)
    results = []
    for gi, g in enumerate(graphs()):
        init = bm.cheap_matching(g)
        pm.upload(g, row_index=(gi % 2 == 0))
        for shortest, kernel, improved in [(False, bm.BfsKernel.GpubfsWr, False), (True, bm.BfsKernel.GpubfsWr, True),
                                           (False, bm.BfsKernel.Gpubfs, False)]:
            res = pm.match(init, shortest=shortest, kernel=kernel, improved=improved)
            m = pm.gather()
            results.append({"graph": gi, "card": res.cardinality, "rmatch": m.rmatch.tolist(),
                            "cmatch": m.cmatch.tolist()})
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(results, f)
    dist.barrier()
    dist.destroy_process_group()
