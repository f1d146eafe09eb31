"""Median kernel time over 5 runs per config (tuning A/B; BM_LIB selects a build)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_1379_b200 as bm
cfgs = sys.argv[1:] or ["C2", "C3", "C4"]
out = {"lib": os.path.basename(os.environ.get("BM_LIB", "default")), "persist": os.environ.get("BM_PERSIST_MB", "0")}
for cfg in cfgs:
    g, known = bench.build_graph(cfg, 1)
    init = bm.cheap_matching(g)
    eng = bm.Engine(0); eng.upload(g); eng.load_matching(init)
    if os.environ.get("PERF_BU") == "1":  # pulled dense levels (AUTO with a prepared row index)
        eng.prepare_row_index()
        eng.bottom_up = True
    eng.run()
    ms, ph, lv, ok = [], [], [], True
    for _ in range(5):
        card, ct, done = eng.run()
        ms.append(eng.last_kernel_time()[0]); ph.append(ct.outer_iterations); lv.append(ct.bfs_launches_total())
        ok = ok and done and (known is None or card == known)
    out[cfg] = {"ms_med": round(statistics.median(ms), 2), "ms": [round(x, 2) for x in ms], "phases": ph, "levels": lv,
                "ms_per_phase": round(sum(ms) / sum(ph), 3), "ok": ok}
    del eng
print(json.dumps(out), flush=True)
