"""Tiny push-only run for compute-sanitizer --tool racecheck (the open racecheck item)."""
import os, sys
sys.path.insert(0, '/root/repo')
import paper_1303_1379_b200 as bm
which = sys.argv[1] if len(sys.argv) > 1 else "tiny"
if which == "tiny":
    g = bm.generate_random_bipartite(3000, 3000, 4.0, 1)
elif which == "uniform":
    g = bm.generate_random_bipartite(200000, 200000, 8.0, 1)
else:
    g = bm.generate_banded(300000, 3, 0.05, 2)[0]
eng = bm.Engine(0)
eng.bottom_up = False
eng.upload(g)
m = eng.match(g, bm.cheap_matching(g)).matching
print("card", bm.cardinality(m), flush=True)
