"""A/B of the WR claim policy (0 = reference, 1 = dead trees stop claiming at discovery): median of 5."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_1379_b200 as bm
for cfg in sys.argv[1:] or ["C2", "C3", "C4"]:
    g, known = bench.build_graph(cfg, 1)
    init = bm.cheap_matching(g)
    eng = bm.Engine(0); eng.upload(g); eng.load_matching(init)
    row = {"cfg": cfg}
    for mode in [0, 1, 0, 1]:
        ms, ph = [], []
        for _ in range(5):
            card, ct, done = eng.run(claim_mode=mode)
            assert done and (known is None or card == known)
            ms.append(eng.last_kernel_time()[0]); ph.append(ct.outer_iterations)
        row.setdefault(f"claim{mode}", []).append((round(statistics.median(ms), 2), round(sum(ms) / sum(ph), 3)))
    print(json.dumps(row), flush=True)
    del eng
