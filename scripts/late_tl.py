"""Per-run trace of the late phases (profiling): kernel ms, then every stage in
order with its duration — late levels as b<entries> (backward) / f<entries>
(forward), late phase ends as L<paths>, full phases as P<roots left>.

usage: python scripts/late_tl.py C5 [--reps 6] [KEY=VAL ...]   (env overrides)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1303_1379_b200 as bm  # noqa: E402


def main():
    args = sys.argv[1:]
    cfg = args.pop(0)
    reps = 6
    while args:
        a = args.pop(0)
        if a == "--reps":
            reps = int(args.pop(0))
        else:
            k, v = a.split("=", 1)
            os.environ[k] = v
    os.environ.setdefault("BM_LATE", "1")
    g, known = bench.build_graph(cfg, 1)
    eng = bm.Engine(0)
    eng.upload(g)
    eng.load_matching(bm.cheap_matching(g))
    eng.prepare_row_index()
    for i in range(reps):
        card, ct, done = eng.run(kernel=bm.BfsKernel.GpubfsWr)
        ms, _ = eng.last_kernel_time()
        tl = eng.timeline()
        prev = tl[0][2]
        items, lvl_us = [], 0.0
        for kind, arg, t in tl[1:]:
            dt = (t - prev) / 1e3
            prev = t
            if kind == "late_level":
                items.append(("b" if arg >> 31 else "f") + str(arg & 0x7FFFFFFF) + ":%.0f" % dt)
            elif kind == "late":
                items.append("L%d:%.0f" % (arg, dt))
            elif kind == "roots":
                items.append("P%d[%.0f]" % (arg, lvl_us + dt))
                lvl_us = 0.0
            elif kind != "level_edges":
                lvl_us += dt
        print("run %d: %.2f ms card %d ok %s phases %d | %s" % (i, ms, card, card == known, ct.outer_iterations,
                                                              " ".join(items)), flush=True)
        print("  stats:", {k: v for k, v in eng.debug_stats().items() if k.startswith("late")}, flush=True)


if __name__ == "__main__":
    main()
