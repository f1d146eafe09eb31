"""Generate golden fixtures from the REFERENCE implementation itself.

Runs only where /root/reference exists (this container): it loads
oracle/_ref/libbmatch_ref.so — the reference's own sources compiled
unmodified by `make ref` — and records its outputs. The fixtures travel with
the repo; nothing at test time reads /root/reference.

usage: python tests/golden/make_golden.py [--large]

Writes:
  corpus.json        acceptance corpus (acceptance.cpp:78-108): per instance the
                     CSC digest, brute-force maximum, first-fit cardinality and
                     the Serial-schedule counters of the 8 registry configs
  steps.json         single-kernel traces (gpubfs / gpubfs_wr / alternate /
                     alternate_wr / fix_matching) on small random states
  known_answers.json larger instances: reference cardinalities (and digests)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from conftest import acceptance_corpus, splitmix64  # noqa: E402
from oracle import Reference  # noqa: E402
import paper_1303_1379_b200 as bm  # noqa: E402

CONFIG_IDS = ["apfb-gpubfs-ct", "apfb-gpubfs-mt", "apfb-wr-ct", "apfb-wr-mt",
              "apsb-gpubfs-ct", "apsb-gpubfs-mt", "apsb-wr-ct", "apsb-wr-mt"]


def corpus(ref):
    out = []
    for g in acceptance_corpus(1000):
        rg = ref.from_csc(g)
        assert ref.lib.ref_check_csr(rg.h) == 0, g.name
        r0, c0 = rg.cheap_matching()
        inst = {"name": g.name, "nc": g.nc, "nr": g.nr, "edges": g.num_edges(), "digest": str(bm.csc_digest(g)),
                "maximum": rg.brute_force_maximum(), "first_fit": int((r0 >= 0).sum()), "runs": {}}
        for algo in CONFIG_IDS:
            # the acceptance corpus sweep uses a 256-thread constant grid (acceptance.cpp:160-166)
            r, c, ct, _ = rg.run(algo, r0, c0, "serial", ct_threads=256)
            assert int((r >= 0).sum()) == inst["maximum"], (g.name, algo)
            inst["runs"][algo] = ct
        out.append(inst)
    return out


def steps(ref):
    """Single-level traces under the Serial schedule (tot = 64 threads)."""
    out = []
    for i in range(60):
        nc = 1 + splitmix64(7 * i + 1) % 120
        nr = 1 + splitmix64(7 * i + 2) % 120
        g = bm.generate_random_bipartite(nc, nr, [1.0, 2.0, 4.0, 8.0][i % 4], 777 + i)
        rg = ref.from_csc(g)
        r0, c0 = rg.cheap_matching()
        wr = i % 2
        improved = 1 if (wr and i % 4 == 1) else 0
        bfs = np.where(c0 > -1, 1, 2).astype(np.int32)
        root = np.where(c0 > -1, 0, np.arange(nc)).astype(np.int32)
        pred = np.full(nr, -1, np.int32)
        r, c = r0.copy(), c0.copy()
        flags = np.array([1, 0], np.int32)
        trace = []
        level = 2
        while flags[0]:
            flags[0] = 0
            p32 = lambda a: a.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_int32))  # noqa: E731
            scans = ref.lib.ref_gpubfs(rg.h, 64, wr, improved, level, p32(bfs), p32(pred), p32(root), p32(r), p32(c),
                                       p32(flags))
            trace.append({"level": level, "scans": int(scans), "bfs": bfs.tolist(), "pred": pred.tolist(),
                          "root": root.tolist() if wr else None, "rmatch": r.tolist(), "flags": flags.tolist()})
            level += 1
        ra, ca = r.copy(), c.copy()
        walks = ref.lib.ref_alternate(rg.h, 64, improved, p32(bfs), p32(pred), p32(ra), p32(ca))
        resets, rf, cf = ref.fix_matching(ra, ca)
        out.append({"nc": nc, "nr": nr, "deg": [1.0, 2.0, 4.0, 8.0][i % 4], "seed": 777 + i, "wr": wr,
                    "improved": improved, "init_rmatch": r0.tolist(), "init_cmatch": c0.tolist(), "levels": trace,
                    "alternate": {"walks": int(walks), "rmatch": ra.tolist(), "cmatch": ca.tolist()},
                    "fix": {"resets": resets, "rmatch": rf.tolist(), "cmatch": cf.tolist()}})
    return out


def known_answers(ref, large):
    ans = {}
    cases = [("uniform", 100_000, 8.0, 1), ("uniform", 200_000, 6.0, 4242), ("uniform", 1_000_000, 8.0, 1)]
    for kind, n, d, s in cases:
        g = bm.generate_random_bipartite(n, n, d, s)
        rg = ref.from_csc(g)
        r0, c0 = rg.cheap_matching()
        r, c, ct, secs = rg.run("apfb-wr-ct", r0, c0, "parallel")
        ans[f"{kind}/{n}/{d}/{s}"] = {"edges": g.num_edges(), "digest": str(bm.csc_digest(g)),
                                      "first_fit": int((r0 >= 0).sum()), "maximum": int((r >= 0).sum()),
                                      "reference_counters": ct}
    # scaled-down versions of the new configs (generator defined in bm_host.cpp)
    for name, g in [("rmat/18/16/2024", bm.generate_rmat(18, 16.0, 2024)),
                    ("rmat/20/16/2024", bm.generate_rmat(20, 16.0, 2024)),
                    ("planted/1000000/16/2024", bm.generate_planted(1_000_000, 16.0, 2024)),
                    ("banded/1000000/3/0.05/12345", bm.generate_banded(1_000_000, 3, 0.05, 12345)[0])]:
        rg = ref.from_csc(g)
        r0, c0 = rg.cheap_matching()
        r, c, ct, secs = rg.run("apfb-wr-ct", r0, c0, "parallel")
        ans[name] = {"edges": g.num_edges(), "digest": str(bm.csc_digest(g)), "first_fit": int((r0 >= 0).sum()),
                     "maximum": int((r >= 0).sum()), "reference_counters": ct}
    if large:
        g = bm.generate_rmat(24, 16.0, 2024)  # C3 at full scale
        rg = ref.from_csc(g)
        r0, c0 = rg.cheap_matching()
        r, c, ct, secs = rg.run("apfb-wr-ct", r0, c0, "parallel")
        ans["C3/div1"] = int((r >= 0).sum())
        ans["rmat/24/16/2024"] = {"edges": g.num_edges(), "digest": str(bm.csc_digest(g)),
                                  "first_fit": int((r0 >= 0).sum()), "maximum": int((r >= 0).sum()),
                                  "reference_counters": ct, "reference_seconds": secs}
    return ans


def main():
    ref = Reference()
    large = "--large" in sys.argv
    with open(os.path.join(HERE, "corpus.json"), "w") as f:
        json.dump(corpus(ref), f, separators=(",", ":"))
    with open(os.path.join(HERE, "steps.json"), "w") as f:
        json.dump(steps(ref), f, separators=(",", ":"))
    path = os.path.join(HERE, "known_answers.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    old.update(known_answers(ref, large))
    with open(path, "w") as f:
        json.dump(old, f, indent=1)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
