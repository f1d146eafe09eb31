"""Phase-1-only kernel time (max_phases=1), median of 7, for builds given as BM_LIB (timing experiments)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_1379_b200 as bm
out = {"lib": os.path.basename(os.environ.get("BM_LIB", "default"))}
for cfg in sys.argv[1:] or ["C2"]:
    g, known = bench.build_graph(cfg, 1)
    init = bm.cheap_matching(g)
    eng = bm.Engine(0); eng.upload(g); eng.load_matching(init)
    ms = []
    for _ in range(8):
        eng.run(max_phases=1)
        ms.append(eng.last_kernel_time()[0])
    out[cfg] = round(statistics.median(ms[1:]), 3)
    del eng
print(json.dumps(out), flush=True)
