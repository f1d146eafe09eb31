"""One matching run limited to the first phase (for profiling the claim-heavy levels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1303_1379_b200 as bm
g, known = bench.build_graph(sys.argv[1] if len(sys.argv) > 1 else "C2", 1)
init = bm.cheap_matching(g)
eng = bm.Engine(0); eng.upload(g); eng.load_matching(init)
for _ in range(3):
    eng.run(max_phases=1)
print(eng.last_kernel_time())
