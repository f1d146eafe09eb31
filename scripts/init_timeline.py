"""Stage timeline of one-call bm_match runs on C5: given first-fit init (validated in the
kernel's setup) against the GPU cheap init (BM_INIT_GPU_KS)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1303_1379_b200 as bm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
g, _ = bench.build_graph(cfg)
init = bm.cheap_matching(g)
eng = bm.Engine(0)
eng.upload(g)
eng.prepare_row_index()
for mode in ("given", "gpu_ks", "gpu_greedy", "given", "gpu_ks"):
    res = eng.match(g, init if mode == "given" else None, init_mode=mode)
    k, _ = eng.last_kernel_time()
    tl = eng.timeline()
    t0 = tl[0][2]
    stages = {}
    prev = t0
    for kind, arg, t in tl[1:]:
        if kind == "level_edges":
            continue
        stages[kind] = stages.get(kind, 0.0) + (t - prev) / 1e6
        prev = t
    print(mode, f"kernel {k:.1f} ms, phases {res.counters.outer_iterations}, init card {res.counters.initial_cardinality}",
          {s: round(v, 2) for s, v in stages.items()}, flush=True)
