"""Pulled-level parity sweep on skewed graphs (debugging aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1303_1379_b200 as bm
from oracle import Oracle
orc = Oracle()
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 14
for alpha in ["4", "1", "14", "100"]:
    os.environ["BM_BU_ALPHA"] = alpha
    g = bm.generate_rmat(scale, 16.0, 2024)
    want = orc.maximum(g)
    init = bm.cheap_matching(g)
    eng = bm.Engine(0)
    eng.upload(g)
    eng.prepare_row_index()
    eng.bottom_up = True
    for algo in [(False, 1, False), (True, 1, True), (False, 0, False)]:
        r = eng.match(g, init, shortest=algo[0], kernel=bm.BfsKernel(algo[1]), improved=algo[2])
        st = eng.debug_stats()
        print(scale, alpha, algo, bm.cardinality(r.matching), want, st.get("pulled_levels"), st.get("materialized"), flush=True)
