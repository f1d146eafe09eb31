"""Host memory copy rate on the GPU box (pageable -> pinned), by thread count:
the ceiling of the staged path that pageable host buffers take (xfer_h2d)."""
import os
import threading
import time

import numpy as np
import torch

n = 1 << 30  # 1 GiB
src = np.ones(n, np.uint8)
dst = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), flush=True)
for t in (1, 2, 4, 8, 12, 16, 24, 32, 48, 64):
    if t > len(os.sched_getaffinity(0)) * 2:
        break
    best = 1e9
    for _ in range(3):
        parts = [(n * i // t, n * (i + 1) // t) for i in range(t)]
        th = [threading.Thread(target=lambda a, b: np.copyto(dst[a:b], src[a:b]), args=pa) for pa in parts]
        t0 = time.perf_counter()
        for x in th:
            x.start()
        for x in th:
            x.join()
        best = min(best, time.perf_counter() - t0)
    print(f"threads {t:3d}: {n / best / 1e9:6.1f} GB/s", flush=True)
