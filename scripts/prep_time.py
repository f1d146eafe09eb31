"""Time bm_prepare_row_index (the row index of the pulled levels) across repeated uploads of C2."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch, bench
import paper_1303_1379_b200 as bm
g, _ = bench.build_graph("C2")
eng = bm.Engine(0)
for rep in range(3):
    t = time.perf_counter(); eng.upload(g, force=True); torch.cuda.synchronize(); tu = time.perf_counter() - t
    t = time.perf_counter(); eng.prepare_row_index(); tp = time.perf_counter() - t
    t = time.perf_counter(); eng.prepare_row_index(); tp2 = time.perf_counter() - t
    print(f"rep {rep} upload {tu*1e3:.1f} ms prepare {tp*1e3:.1f} ms again {tp2*1e3:.2f} ms", flush=True)
