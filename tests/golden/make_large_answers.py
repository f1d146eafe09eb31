"""Full-size known answers computed by the REFERENCE (oracle/_ref, its own sources
compiled unmodified): the maximum-matching cardinality of configs C3 and C4 as
built by this repo's generators, and a digest of each graph so a generator
change is caught. Runs here (CPU, minutes); the output is committed and read
by the -m gpu full-size parity test (tests/test_full_size.py).

usage: python tests/golden/make_large_answers.py [C3] [C4] [C2]
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1303_1379_b200 as bm  # noqa: E402
from oracle import Reference  # noqa: E402


def main():
    cfgs = sys.argv[1:] or ["C3", "C4"]
    ref = Reference()
    path = os.path.join(HERE, "known_answers.json")
    ans = json.load(open(path))
    for cfg in cfgs:
        g, known = bench.build_graph(cfg, 1)
        rg = ref.from_csc(g)
        r0, c0 = rg.cheap_matching()
        t = time.perf_counter()
        r, c, ct, secs = rg.run("apfb-wr-ct", r0, c0, "parallel")
        card = int((r >= 0).sum())
        if known is not None:
            assert card == known, (cfg, card, known)
        ans[f"{cfg}/div1"] = card
        ans[f"{cfg}/full"] = {"edges": g.num_edges(), "digest": str(bm.csc_digest(g)), "first_fit": int((r0 >= 0).sum()),
                              "maximum": card, "reference": "apfb-wr-ct parallel", "reference_seconds": secs}
        print(cfg, card, f"{time.perf_counter() - t:.1f}s", flush=True)
        del rg
    with open(path, "w") as f:
        json.dump(ans, f, indent=1)


if __name__ == "__main__":
    main()
