"""Small runs with late phases forced on every phase, for compute-sanitizer
(memcheck / racecheck / synccheck): default and tight bounds, square and
rectangular graphs, from first-fit and from the unmatched state, checked
against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BM_LATE", "1")
os.environ.setdefault("BM_LATE_ROOTS", "2000000000")
import paper_1303_1379_b200 as bm  # noqa: E402
import oracle  # noqa: E402

orc = oracle.Oracle()
eng = bm.Engine(0)
eng.bottom_up = True
bad = 0
for g in [bm.generate_random_bipartite(6000, 5000, 4.0, 1), bm.generate_random_bipartite(5000, 6000, 3.0, 2),
          bm.generate_planted(6000, 6.0, 3), bm.generate_rmat(12, 8.0, 3)]:
    want = orc.maximum(g)
    for init in [bm.cheap_matching(g), None]:
        m = eng.match(g, init).matching
        st = eng.debug_stats()
        ok = bm.cardinality(m) == want and orc.validate(g, m.rmatch, m.cmatch) == 0
        bad += 0 if ok else 1
        print(g.nc, g.nr, g.num_edges(), bm.cardinality(m), want, "ok" if ok else "MISMATCH",
              {k: v for k, v in st.items() if k.startswith("late")}, flush=True)
print("late sanitize run:", "PASS" if bad == 0 else f"{bad} FAIL")
