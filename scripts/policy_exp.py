"""Experiment: WR claim x endpoint policy vs phases / traversed edges / kernel time."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_1379_b200 as bm
cfgs = sys.argv[1:] or ["C2", "C3", "C4", "C1"]
for cfg in cfgs:
    g, known = bench.build_graph(cfg, 1)
    init = bm.cheap_matching(g)
    eng = bm.Engine(0); eng.upload(g); eng.load_matching(init)
    for algo in ["apfb-wr", "apsb-wr"]:
        sh, k, imp = bench.ALGOS[algo]
        for mode in [0, 1]:
            for ep in [1, 2]:
                res = []
                for rep in range(3):
                    card, ct, done = eng.run(shortest=sh, kernel=bm.BfsKernel(k), improved=imp, claim_mode=mode,
                                             endpoint_policy=ep)
                    ms, _ = eng.last_kernel_time()
                    unmatched = [a for kind, a, t in eng.timeline() if kind == "roots"]
                    ok = (known is None or card == known) and done
                    res.append((round(ms, 2), ct.outer_iterations, ct.bfs_launches_total(), ct.edges_traversed,
                                ct.columns_visited, ct.alternations_attempted, ct.fix_resets, ok, unmatched[:12]))
                print(json.dumps({"cfg": cfg, "algo": algo, "claim": mode, "ep": ep, "card": card, "runs": res}),
                      flush=True)
