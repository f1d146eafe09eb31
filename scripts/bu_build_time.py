"""Time the row-index (transpose) build that the pulled levels need.

usage: python scripts/bu_build_time.py C2
Prints the first bottom-up run (which builds the index) against later runs.
"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1303_1379_b200 as bm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
g, _ = bench.build_graph(cfg)
init = bm.cheap_matching(g)
eng = bm.Engine(0)
out = {"config": cfg}
for rep in range(2):
    t = time.perf_counter()
    eng.upload(g, force=True)
    torch.cuda.synchronize()
    out[f"upload_s_{rep}"] = time.perf_counter() - t
    eng.load_matching(init)
    t = time.perf_counter()
    eng.run(bottom_up=True)
    torch.cuda.synchronize()
    out[f"first_bu_run_s_{rep}"] = time.perf_counter() - t
    t = time.perf_counter()
    eng.run(bottom_up=True)
    torch.cuda.synchronize()
    out[f"second_bu_run_s_{rep}"] = time.perf_counter() - t
print(json.dumps(out))
