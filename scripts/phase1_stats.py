"""CTA-cycle split of the first phase only (claim-heavy levels) for C2."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_1379_b200 as bm
g, known = bench.build_graph(sys.argv[1] if len(sys.argv) > 1 else "C2", 1)
init = bm.cheap_matching(g)
eng = bm.Engine(0); eng.upload(g); eng.load_matching(init)
for mp in [1, 2, 0]:
    for rep in range(2):
        card, ct, done = eng.run(max_phases=mp)
        ms, _ = eng.last_kernel_time()
    ds = eng.debug_stats()
    cyc = {k: v for k, v in ds.items() if k.startswith("cyc")}
    tot = sum(cyc.values())
    print(json.dumps({"max_phases": mp, "ms": round(ms, 3), "split": {k: round(v / tot, 3) for k, v in cyc.items()},
                      "cta_ms": round(tot / 592 / 1.965e6, 3), "claims": ds["columns_visited"], "edges": ds["edges_traversed"],
                      "entries": ds["frontier_entries"]}))
