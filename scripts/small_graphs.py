"""Wall vs kernel time of one-shot matches on the suite's small instances."""
import sys, time
sys.path.insert(0, '/root/repo')
import paper_1303_1379_b200 as bm
for n, d in [(200000, 4.0), (1000000, 3.0), (500000, 8.0)]:
    g = bm.generate_random_bipartite(n, n, d, 1 if d == 4.0 else 3 if d == 3.0 else 2)
    init = bm.cheap_matching(g)
    eng = bm.Engine(0)
    for rep in range(3):
        t = time.perf_counter(); r = eng.match(g, init); t = time.perf_counter() - t
    kms, nl = eng.last_kernel_time()
    c = r.counters
    print(n, d, f"wall {t*1e3:.2f} ms kernel {kms:.2f} ms phases {c.outer_iterations} levels {c.bfs_launches_total()} card {bm.cardinality(r.matching)}", flush=True)
