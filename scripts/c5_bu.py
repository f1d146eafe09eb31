"""C5 at full size: push-only vs bottom-up dense levels (median of 3), and the row-index build time."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_1379_b200 as bm
g, known = bench.build_graph("C5", 1)
init = bm.cheap_matching(g)
eng = bm.Engine(0); eng.upload(g); eng.load_matching(init)
out = {}
for bu in [False, True]:
    t = time.perf_counter(); card, ct, done = eng.run(bottom_up=bu); t = time.perf_counter() - t
    ms = []
    ph = []
    for _ in range(3):
        card, ct, done = eng.run(bottom_up=bu)
        ms.append(eng.last_kernel_time()[0]); ph.append(ct.outer_iterations)
    out["bottom_up" if bu else "push"] = {"ms": [round(x, 1) for x in ms], "phases": ph, "first_call_s": round(t, 3),
                                          "card": card, "ok": done and card == known,
                                          "edges_traversed": ct.edges_traversed}
print(json.dumps(out))
