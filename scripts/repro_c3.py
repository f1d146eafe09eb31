"""Full-size C3 with pulled levels, repeated under env variants (debugging aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_1303_1379_b200 as bm
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
specs = sys.argv[3:] or ["-"]
g, known = bench.build_graph(cfg, 1)
known = known or bench.known_answers().get(f"{cfg}/div1")
init = bm.cheap_matching(g)
base = dict(os.environ)
for spec in specs:
    os.environ.clear(); os.environ.update(base)
    if spec != "-":
        for kv in spec.split(","):
            k, v = kv.split("=", 1); os.environ[k] = v
    fails, oks = [], 0
    for r in range(reps):
        eng = bm.Engine(0)
        eng.upload(g)
        eng.load_matching(init)
        eng.prepare_row_index()
        for algo in ["apfb-wr", "apsb-wr", "apfb-gpubfs"]:
            s, k, imp = bench.ALGOS[algo]
            try:
                card, ct, done = eng.run(shortest=s, kernel=bm.BfsKernel(k), improved=imp, bottom_up=True)
                oks += card == known
            except Exception as e:
                fails.append((algo, str(e)[-120:]))
                eng = bm.Engine(0); eng.upload(g); eng.load_matching(init); eng.prepare_row_index()
    print(spec, "ok", oks, "fails", len(fails), fails[:3], flush=True)
