"""Upload / match / download times from pinned and from pageable host arrays
(the staged path), C2 or C5: where the pageable e2e loses its time."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1303_1379_b200 as bm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
g, _ = bench.build_graph(cfg)
init = bm.cheap_matching(g)
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
gp = bm.BipartiteCsr(g.nc, g.nr, pin(g.cxadj), pin(g.cadj), g.name)
eng = bm.Engine(0)
for name, gg, mk in [("pinned", gp, lambda: bm.MatchingState(pin(init.rmatch), pin(init.cmatch))),
                     ("pageable", g, lambda: init.copy())]:
    up, mt, tot = [], [], []
    for i in range(5):
        m = mk()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.upload(gg, force=True)
        t1 = time.perf_counter()
        eng.match_inplace(gg, m)
        t2 = time.perf_counter()
        if i:
            up.append(1e3 * (t1 - t0)); mt.append(1e3 * (t2 - t1)); tot.append(1e3 * (t2 - t0))
    k, _ = eng.last_kernel_time()
    print(f"{cfg} {name:9s} upload {statistics.median(up):7.1f} ms  match(+init H2D, D2H) {statistics.median(mt):7.1f} ms"
          f"  total {statistics.median(tot):7.1f} ms  (kernel {k:.1f} ms)", flush=True)
