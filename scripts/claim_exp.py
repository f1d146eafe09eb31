"""Experiment: WR claim policy vs phases / traversed edges / time (per-phase unmatched counts)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_1379_b200 as bm
for cfg, div in [("C2", 10), ("C2", 1), ("C1", 1), ("C3", 1)]:
    g, known = bench.build_graph(cfg, div)
    init = bm.cheap_matching(g)
    eng = bm.Engine(0); eng.upload(g); eng.load_matching(init)
    for algo in ["apfb-wr", "apfb-gpubfs", "apsb-wr"]:
        sh, k, imp = bench.ALGOS[algo]
        modes = [0, 1] if k == 1 else [0]
        for mode in modes:
            res = []
            for rep in range(3):
                card, ct, done = eng.run(shortest=sh, kernel=bm.BfsKernel(k), improved=imp, claim_mode=mode)
                ms, _ = eng.last_kernel_time()
                tl = eng.timeline()
                unmatched = [a for kind, a, t in tl if kind == "roots"]
                res.append((round(ms, 2), ct.outer_iterations, ct.edges_traversed, ct.columns_visited, unmatched))
            print(json.dumps({"cfg": cfg, "div": div, "algo": algo, "mode": mode, "runs": res}))
