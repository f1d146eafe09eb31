"""Push-only runs for compute-sanitizer --tool racecheck (the push-path racecheck item).

usage: [BM_GRID_CTAS=1] compute-sanitizer --tool racecheck python scripts/racecheck_push.py tiny|uniform|banded
BM_GRID_CTAS=1 runs the persistent kernel as a single CTA: every grid barrier
returns at once (the CTA is its own last arriver), so the run has no
cross-CTA spinning while the window scan, rounds and flushes of expand_level
execute exactly as in a full grid (every tile and window, one CTA after another).
"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_1379_b200 as bm  # noqa: E402
from oracle import Oracle  # noqa: E402

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
want = Oracle().maximum(g)
print("card", bm.cardinality(m), "oracle", want, "ok", bm.cardinality(m) == want, flush=True)
