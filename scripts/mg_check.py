"""Multi-GPU engine on one device: teams of 1-4 ranks in this process (one
stream each) against the oracle's maxima, then C2/C5 team-of-1 timing against
the single-GPU engine. usage: python scripts/mg_check.py [quick|C2|C5 ...]"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1303_1379_b200 as bm  # noqa: E402
from paper_1303_1379_b200.partition import LocalTeam  # noqa: E402


def parity():
    from oracle import Oracle
    from conftest import acceptance_corpus
    orc = Oracle()
    gs = acceptance_corpus(24)
    gs += [bm.generate_random_bipartite(3000, 2500, 3.0, 41), bm.generate_planted(2000, 4.0, 5),
           bm.generate_banded(3000, 3, 0.05, 9)[0], bm.generate_rmat(11, 8.0, 3),
           bm.generate_random_bipartite(200000, 200000, 6.0, 4242)]
    bad = 0
    for world in (1, 2, 3, 4):
        for ri in (False, True):
            team = LocalTeam(world)
            for gi, g in enumerate(gs):
                init = bm.cheap_matching(g)
                want = orc.maximum(g)
                team.upload(g, row_index=ri)
                for shortest, kernel, improved in [(False, bm.BfsKernel.GpubfsWr, False),
                                                   (True, bm.BfsKernel.GpubfsWr, True),
                                                   (False, bm.BfsKernel.Gpubfs, False)]:
                    res, m = team.match(init, shortest=shortest, kernel=kernel, improved=improved,
                                        bottom_up="on" if ri else "off")
                    ok = (res.cardinality == want and bm.cardinality(m) == want
                          and orc.validate(g, m.rmatch, m.cmatch) == 0 and orc.is_maximum(g, m.rmatch, m.cmatch) == 1)
                    if not ok:
                        bad += 1
                        print("FAIL", world, ri, gi, g.nc, g.nr, shortest, int(kernel), res.cardinality,
                              bm.cardinality(m), want, flush=True)
            team.close()
            print(f"world {world} row_index {ri}: done, failures so far {bad}", flush=True)
    return bad


def timing(cfg, worlds=(1, 2)):
    import bench
    g, known = bench.build_graph(cfg)
    if known is None:
        known = bench.known_answers().get(f"{cfg}/div1")
    init = bm.cheap_matching(g)
    eng = bm.Engine(0)
    eng.upload(g)
    eng.load_matching(init)
    eng.prepare_row_index()
    single = []
    for _ in range(4):
        card, ct, done = eng.run(bottom_up="auto")
        single.append(eng.last_kernel_time()[0])
    eng.close()
    print(f"{cfg} single-GPU engine: {statistics.median(single[1:]):.2f} ms (card {card})", flush=True)
    for world in worlds:
        team = LocalTeam(world)
        t = time.perf_counter()
        team.upload(g, row_index=True)
        t = time.perf_counter() - t
        for bu in ("auto", "off"):
            ms, ph = [], []
            for _ in range(4):
                res, m = team.match(init, bottom_up=bu)
                ms.append(res.kernel_ms)
                ph.append(res.phases)
            ok = known is None or res.cardinality == known
            print(f"{cfg} team of {world} on one GPU, bottom_up={bu}: {statistics.median(ms[1:]):.2f} ms "
                  f"(phases {ph}, card {res.cardinality}, ok {ok}; setup {t:.1f} s)", flush=True)
        team.close()


if __name__ == "__main__":
    args = sys.argv[1:] or ["quick"]
    rc = 0
    for a in args:
        if a == "quick":
            rc |= 1 if parity() else 0
        else:
            timing(a)
    sys.exit(rc)
