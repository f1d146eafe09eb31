"""Worker for the multi-rank partition tests (spawned with torch.multiprocessing).

Each rank builds the same graphs, runs the partitioned driver with the given
backend ("cpu": the oracle restatement, gloo on host tensors; "gpu": the
bm_part_* kernels on cuda:0, records exchanged with gloo through host memory,
or NCCL when one GPU per rank is available) and saves its results."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def graphs():
    import paper_1303_1379_b200 as bm
    from conftest import acceptance_corpus, fork_graph
    gs = acceptance_corpus(24)  # small random corpus + empty, edgeless, complete, fork
    gs.append(bm.generate_random_bipartite(3000, 2500, 3.0, 41))
    gs.append(bm.generate_planted(2000, 4.0, 5))
    g, _ = bm.generate_banded(3000, 3, 0.05, 9)
    gs.append(g)
    gs.append(bm.generate_rmat(11, 8.0, 3))
    return gs


def run(rank, world, port, backend, out_dir, device_mode):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl" if device_mode == "nccl" else "gloo", rank=rank, world_size=world)
    # "p2p": the fused exchange through CUDA IPC peer memory (gloo only carries the setup and the
    # per-phase broadcast); with several ranks on one GPU the "peers" are the same device
    import paper_1303_1379_b200 as bm
    from paper_1303_1379_b200.partition import Exchange, GpuPartition, PartitionedMatcher
    if backend == "cpu":
        from oracle.partition_ref import CpuPartition
        be = CpuPartition(rank, world)
    else:
        dev = rank if device_mode == "nccl" else 0
        torch.cuda.set_device(dev)
        be = GpuPartition(dev, rank, world)
    pm = PartitionedMatcher(be, Exchange())
    results = []
    for gi, g in enumerate(graphs()):
        init = bm.cheap_matching(g)
        pm.upload(g, p2p=(device_mode == "p2p"))
        for shortest, kernel in [(False, bm.BfsKernel.GpubfsWr), (True, bm.BfsKernel.GpubfsWr),
                                 (False, bm.BfsKernel.Gpubfs)]:
            res = pm.match(init, shortest=shortest, kernel=kernel)
            rm, cm = be.state()
            m = bm.MatchingState(rm[:g.nr].cpu().numpy().copy(), cm[:g.nc].cpu().numpy().copy())
            results.append({"graph": gi, "shortest": shortest, "kernel": int(kernel), "card": res.cardinality,
                            "phases": res.phases, "levels": res.levels, "retries": res.serial_retries,
                            "rmatch": m.rmatch.tolist(), "cmatch": m.cmatch.tolist()})
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(results, f)
    dist.barrier()
    dist.destroy_process_group()
