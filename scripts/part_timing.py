"""Host-side stage timing of the partitioned driver at world 1 (NCCL) on C2."""
import json, os, sys, time
os.environ["BM_PART_TIMING"] = "1"
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29577")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import bench
import paper_1303_1379_b200 as bm
from paper_1303_1379_b200.partition import Exchange, GpuPartition, PartitionedMatcher
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
g, known = bench.build_graph(sys.argv[1] if len(sys.argv) > 1 else "C2", 1)
init = bm.cheap_matching(g)
pm = PartitionedMatcher(GpuPartition(0, 0, 1), Exchange())
pm.upload(g, p2p=os.environ.get("BM_P2P") == "1")
pm.match(init)
pm.t = {}
t = time.perf_counter(); r = pm.match(init); t = time.perf_counter() - t
print(json.dumps({"ms": t * 1e3, "card": r.cardinality, "phases": r.phases, "levels": r.levels,
                  "stages_ms": {k: round(v * 1e3, 2) for k, v in pm.t.items()}}))
dist.destroy_process_group()
