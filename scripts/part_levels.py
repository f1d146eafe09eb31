"""Per-level frontier sizes of the partitioned engine (world 1) vs the single-GPU engine on the same graph."""
import json, os, sys
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29581")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import bench
import paper_1303_1379_b200 as bm
from paper_1303_1379_b200.partition import Exchange, GpuPartition, PartitionedMatcher
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
g, known = bench.build_graph(sys.argv[1] if len(sys.argv) > 1 else "C2", int(sys.argv[2]) if len(sys.argv) > 2 else 1)
init = bm.cheap_matching(g)
be = GpuPartition(0, 0, 1)
pm = PartitionedMatcher(be, Exchange())
pm.upload(g)
# instrument: record n_cur and record counts per level
orig_expand = be.expand
log = []
def expand():
    c, e, a, b = orig_expand()
    log.append((be._n_cur_dbg() if hasattr(be, "_n_cur_dbg") else None, a, b))
    return c, e, a, b
be.expand = expand
r = pm.match(init)
st = be.stats()
eng = bm.Engine(0); eng.upload(g); eng.load_matching(init)
card, ct, done = eng.run()
tl = eng.timeline()
lv = [(a, t) for (k, a, t) in tl if k == "level"]
print(json.dumps({"partition": {"phases": r.phases, "levels": r.levels, "stats": st,
                                "claims_per_level": [x[1] for x in log][:30], "eps_per_level": [x[2] for x in log][:30]},
                  "single": {"phases": ct.outer_iterations, "edges_traversed": ct.edges_traversed,
                             "columns_scanned": ct.columns_scanned, "columns_visited": ct.columns_visited,
                             "entries_per_level": [a for a, t in lv][:30]}}))
dist.destroy_process_group()
