"""A/B the pull rule and lazy-frontier knobs on one resident graph (profiling).

usage: python scripts/tune.py C5 [--div N] [--reps 3] [--tl] KEY=VAL[,KEY=VAL...] ...
Each positional spec is a set of env overrides (BM_BU_ALPHA=8,BM_BU_BETA=24);
"-" is the defaults. Prints one JSON line per spec: kernel ms (min/median),
phases, levels, pulled levels, cardinality check; --tl adds the per-level timeline
of the last run of every spec.
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1303_1379_b200 as bm  # noqa: E402


def timeline_summary(eng):
    tl = eng.timeline()
    levels, prev = [], tl[0][2]
    phase = 0
    kinds = {}
    sub = {}
    for kind, arg, t in tl[1:]:
        if kind == "level_edges":
            levels[-1] += [arg & 0x7FFFFFFF, arg >> 31]
            continue
        dt = (t - prev) / 1e3
        prev = t
        kinds[kind] = kinds.get(kind, 0.0) + dt
        if kind in ("materialize", "pull_prep", "bucketed"):  # parts of the level that follows
            sub[kind] = round(dt, 1)
            continue
        if kind == "level":
            levels.append([phase, arg, round(dt + sum(sub.values()), 1), sub])
            sub = {}
        if kind == "roots":
            phase += 1
    return {"per_kind_us": {k: round(v, 1) for k, v in kinds.items()}, "levels": levels}


def main():
    args = sys.argv[1:]
    cfg = args.pop(0)
    div, reps, tl, algo = 1, 3, False, "apfb-wr"
    specs = []
    while args:
        a = args.pop(0)
        if a == "--div":
            div = int(args.pop(0))
        elif a == "--reps":
            reps = int(args.pop(0))
        elif a == "--tl":
            tl = True
        elif a == "--algo":
            algo = args.pop(0)
        else:
            specs.append(a)
    specs = specs or ["-"]
    g, known = bench.build_graph(cfg, div)
    if known is None:
        known = bench.known_answers().get(f"{cfg}/div{div}")
    init = bm.cheap_matching(g)
    eng = bm.Engine(0)
    eng.upload(g)
    eng.load_matching(init)
    eng.prepare_row_index()
    shortest, kernel, improved = bench.ALGOS[algo]
    base_env = dict(os.environ)
    for spec in specs:
        os.environ.clear()
        os.environ.update(base_env)
        if spec != "-":
            for kv in spec.split(","):
                k, v = kv.split("=", 1)
                os.environ[k] = v
        bu = os.environ.get("TUNE_BU", "auto")
        bu = {"auto": "auto", "on": True, "off": False}[bu]
        ms, phases, levels, cards = [], [], [], []
        for _ in range(reps + 1):
            card, ct, done = eng.run(shortest=shortest, kernel=bm.BfsKernel(kernel), improved=improved,
                                     bottom_up=bu)
            k_ms, _ = eng.last_kernel_time()
            ms.append(k_ms)
            phases.append(ct.outer_iterations)
            levels.append(ct.bfs_launches_total())
            cards.append(card)
        ms = ms[1:]
        st = eng.debug_stats()
        out = {"spec": spec, "cfg": cfg, "algo": algo, "ms_min": round(min(ms), 2),
               "ms_med": round(statistics.median(ms), 2), "ms": [round(x, 2) for x in ms],
               "phases": phases[1:], "levels": levels[1:], "ok": all(c == known for c in cards) if known else None,
               "card": cards[-1], "edges_traversed": ct.edges_traversed, "columns_scanned": ct.columns_scanned,
               "stats": {k: st.get(k) for k in ("rows_pulled", "pulled_levels", "materialized", "cyc_bu_screen", "cyc_bu_probe", "cyc_bu_flush", "bu_rounds", "cyc_tile", "cyc_window", "cyc_rounds", "cyc_flush", "cyc_barrier")}}
        if tl:
            out["timeline"] = timeline_summary(eng)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
