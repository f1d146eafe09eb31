import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_1379_b200 as bm
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
div = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g, known = bench.build_graph(cfg, div)
init = bm.cheap_matching(g)
eng = bm.Engine(0); eng.upload(g); eng.load_matching(init)
card, ct, done = eng.run()
print("card", card, "known", known, "done", done, ct.outer_iterations)
