"""CPU restatement of the partitioned driver's device backend — TEST
INFRASTRUCTURE ONLY (the checker for paper_1303_1379_b200/partition.py; never
the product path).

It implements the same per-rank operations as bm_partition.cu (begin_phase /
expand / merge / end_bfs / augment) sequentially in numpy, with the same
record formats and the same merge rule (lowest (rank, index) record wins per
column, per root and per free row), so the world-size > 1 host protocol can be
run with gloo on CPU. The level and ALTERNATE/FIX semantics follow the
reference: gpubfs / gpubfs_wr gpu_match.cpp:42-70, 99-133; alternate_walk
gpu_match.cpp:144-154; fix_matching gpu_match.cpp:220-245.
"""
from __future__ import annotations

import numpy as np
import torch

VIS = 1 << 30
INT_MAX = np.iinfo(np.int32).max


class CpuPartition:
    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world
        self.st = np.zeros(5, np.int64)  # edges, cols, walks, steps, resets

    def upload(self, nc, nr, lo, hi, cxs, adjs):
        self.nc, self.nr, self.lo, self.hi = nc, nr, lo, hi
        self.offs = np.asarray(cxs, np.int64)
        self.adj = np.asarray(adjs, np.int32)
        self.rmatch = torch.zeros(max(nr, 1), dtype=torch.int32)
        self.cmatch = torch.zeros(max(nc, 1), dtype=torch.int32)
        self.pred = np.full(max(nr, 1), -1, np.int32)
        cap = max(1, min(nc, len(self.adj)))
        self.claims = torch.zeros((cap, 4), dtype=torch.int32)
        self.eps = torch.zeros((max(1, min(nr, len(self.adj))), 4), dtype=torch.int32)

    def load(self, m):
        self.rmatch[:self.nr] = torch.from_numpy(np.asarray(m.rmatch, np.int32))
        self.cmatch[:self.nc] = torch.from_numpy(np.asarray(m.cmatch, np.int32))

    def reset_stats(self):
        self.st[:] = 0

    def stats(self):
        d = dict(zip(["edges_traversed", "columns_scanned", "walks", "walk_steps", "fix_resets"],
                     (int(x) for x in self.st)))
        d["launches"] = 0  # no device kernels in the CPU restatement
        return d

    def state(self):
        return self.rmatch, self.cmatch

    def begin_phase(self, kernel, endpoint_policy):
        self.wr = kernel == 1
        self.ep_one = self.wr and endpoint_policy != 1
        self.dead = np.zeros(self.nc, bool)
        self.ep_list = []
        self.found = False
        cm = self.cmatch.numpy()
        self.F = [(c, c) for c in range(self.lo, self.hi)
                  if cm[c] < 0 and self.offs[c - self.lo + 1] > self.offs[c - self.lo]]
        return len(self.F)

    def expand(self):
        rm = self.rmatch.numpy()
        claims, eps = [], []
        for c, root in self.F:
            if self.wr and self.dead[root]:
                continue
            b, e = self.offs[c - self.lo], self.offs[c - self.lo + 1]
            self.st[0] += e - b
            self.st[1] += 1
            for j in range(b, e):
                row = int(self.adj[j])
                cm = int(rm[row])
                if cm >= 0:
                    if not cm & VIS:
                        rm[row] = cm | VIS
                        claims.append((cm, c, root, row))
                elif cm == -1:
                    if self.ep_one and self.dead[root]:
                        continue
                    rm[row] = -2
                    eps.append((row, c, root, 0))
        for buf, recs in ((self.claims, claims), (self.eps, eps)):
            if recs:
                buf[:len(recs)] = torch.tensor(recs, dtype=torch.int32)
        return self.claims, self.eps, len(claims), len(eps)

    @staticmethod
    def _records(all_, counts, stride):
        a = all_.numpy()
        for r in range(len(counts)):
            for k in range(int(counts[r])):
                yield r * stride + k, a[r * stride + k]

    def merge(self, claims_all, claim_counts, cstride, eps_all, ep_counts, estride):
        rm = self.rmatch.numpy()
        # endpoints: lowest record per live root (ONE_PER_TREE), then lowest per row
        win_r, win_e = {}, {}
        recs = list(self._records(eps_all, ep_counts, estride))
        for i, (row, c, root, _) in recs:
            if self.ep_one and not self.dead[root]:
                win_r.setdefault(root, i)
        for i, (row, c, root, _) in recs:
            if (not self.ep_one) or win_r.get(root) == i:
                win_e.setdefault(row, i)
        for i, (row, c, root, _) in recs:
            w = win_e.get(row)
            if w == i:
                rm[row] = -2
                self.pred[row] = c
                if self.wr:
                    self.dead[root] = True
                if self.rank == 0:
                    self.ep_list.append(int(row))
                self.found = True
            elif w is None:
                rm[row] = -1
        # claims: lowest record per column
        win_c = {}
        recs = list(self._records(claims_all, claim_counts, cstride))
        for i, (cm, c, root, row) in recs:
            win_c.setdefault(cm, i)
        nxt, live = [], 0
        for i, (cm, c, root, row) in recs:
            if win_c[cm] != i:
                continue
            rm[row] = cm | VIS
            self.pred[row] = c
            if self.wr and self.dead[root]:
                continue
            live += 1
            if self.lo <= cm < self.hi:
                nxt.append((int(cm), int(root)))
        self.F = nxt
        return live, self.found

    def end_bfs(self):
        rm = self.rmatch.numpy()
        m = (rm >= 0) & ((rm & VIS) != 0)
        rm[m] &= ~VIS

    def augment(self, serial):
        rm, cmt = self.rmatch.numpy(), self.cmatch.numpy()
        for row in self.ep_list:  # alternate_walk, gpu_match.cpp:144-154
            self.st[2] += 1
            while row != -1:
                col = int(self.pred[row])
                if col < 0:
                    break
                mr = int(cmt[col])
                if mr >= 0 and self.pred[mr] == col:
                    break
                cmt[col] = row
                rm[row] = col
                row = mr
                self.st[3] += 1
        for r in range(self.nr):  # fix_matching rules 1, 2
            v = rm[r]
            if v == -2 or (v >= 0 and cmt[v] != r):
                rm[r] = -1
                self.st[4] += 1
        for c in range(self.nc):  # rule 3
            r = cmt[c]
            if r >= 0 and rm[r] != c:
                cmt[c] = -1
                self.st[4] += 1
        return int((rm[:self.nr] >= 0).sum())

    def cardinality(self):
        return int((self.rmatch.numpy()[:self.nr] >= 0).sum())
