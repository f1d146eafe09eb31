"""Small pulled-level run for compute-sanitizer (memcheck / synccheck):
every level pulled, the row index built by the bucketed kernels, checked
against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BM_BU_AUTO", "1")
os.environ.setdefault("BM_BU_FRAC", "0")
os.environ.setdefault("BM_SOLO_EDGES", "0")
import paper_1303_1379_b200 as bm  # noqa: E402
import oracle  # noqa: E402

orc = oracle.Oracle()
eng = bm.Engine(0)
for g in [bm.generate_random_bipartite(6000, 5000, 6.0, 1), bm.generate_rmat(12, 8.0, 3),
          bm.generate_banded(5000, 3, 0.1, 4)[0]]:
    eng.upload(g, force=True)
    m = eng.match(g, bm.cheap_matching(g)).matching
    want = orc.maximum(g)
    print(g.nc, g.num_edges(), bm.cardinality(m), want, "ok" if bm.cardinality(m) == want else "MISMATCH", flush=True)
