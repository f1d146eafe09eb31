"""Per-stage device timeline of one matching run (bm_timeline), for profiling.

usage: python scripts/timeline.py [C1|C2|C3|C4|C5] [apfb-wr|apsb-wr|...] [--div N] [--bu]
Prints the time spent per stage kind, per phase, and the slowest BFS levels.
"""
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1303_1379_b200 as bm  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    algo = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "apfb-wr"
    div = int(sys.argv[sys.argv.index("--div") + 1]) if "--div" in sys.argv else 1
    bu = True if "--bu" in sys.argv else (False if "--push" in sys.argv else "auto")  # default: AUTO, as bench.py

    g, known = bench.build_graph(cfg, div)
    init = bm.cheap_matching(g)
    shortest, kernel, improved = bench.ALGOS[algo]
    eng = bm.Engine(0)
    eng.upload(g)
    eng.load_matching(init)
    if bu == "auto":
        eng.prepare_row_index()  # as bench.py: qualifying graphs pull their dense levels
    for _ in range(2):
        eng.run(shortest=shortest, kernel=bm.BfsKernel(kernel), improved=improved, bottom_up=bu)
    card, ct, done = eng.run(shortest=shortest, kernel=bm.BfsKernel(kernel), improved=improved, bottom_up=bu)
    ms, _ = eng.last_kernel_time()
    tl = eng.timeline()
    dstats = eng.debug_stats()
    per_kind = defaultdict(float)
    levels = []
    phases = []
    cur_phase = defaultdict(float)
    prev_t = tl[0][2]
    for kind, arg, t in tl[1:]:
        if kind == "level_edges":  # metadata of the level just recorded: frontier edges, pulled?
            levels[-1] = levels[-1] + (arg & 0x7FFFFFFF, arg >> 31)
            continue
        dt = (t - prev_t) / 1e3  # us
        prev_t = t
        per_kind[kind] += dt
        cur_phase[kind] += dt
        if kind == "level":
            levels.append((len(phases), arg, dt))
        if kind in ("roots", "late"):  # a full phase's or a late phase's end
            phases.append(dict(cur_phase))
            cur_phase = defaultdict(float)
    total = (tl[-1][2] - tl[0][2]) / 1e3
    out = {
        "config": cfg, "algo": algo, "cardinality": card, "known": known, "kernel_ms": ms,
        "timeline_total_us": total, "per_kind_us": {k: round(v, 1) for k, v in per_kind.items()},
        "n_levels": len(levels), "n_phases": len(phases),
        "per_phase_us": [{k: round(v, 1) for k, v in ph.items()} for ph in phases],
        "slowest_levels_us": sorted(levels, key=lambda x: -x[2])[:12],
        "levels_us": [round(x[2], 1) for x in levels],
        "levels_detail": [(x[0], x[1], x[3] if len(x) > 3 else None, x[4] if len(x) > 4 else None, round(x[2], 1))
                          for x in levels],
        "pulled_levels_us": round(sum(x[2] for x in levels if len(x) > 4 and x[4]), 1),
        "bottom_up": bu,
        "counters": {k: getattr(ct, k) for k in ["outer_iterations", "columns_scanned", "edges_traversed",
                                                 "columns_visited", "walk_steps", "alternations_attempted",
                                                 "fix_resets", "frontier_entries"]},
        "launches_per_phase": ct.bfs_launches_per_iteration,
        "debug_stats": dstats,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
