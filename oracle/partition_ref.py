"""CPU stand-in for one rank of the multi-GPU engine — TEST INFRASTRUCTURE
ONLY (the checker for the host protocol in paper_1303_1379_b200/partition.py;
never the product path).

It implements GpuRank's operations (upload / export / import_ / row index /
load / launch / finish / download) on the host so that the world-size > 1
protocol runs over gloo on CPU. What the device does through peer memory —
every rank reading and writing every other rank's slice of the state during
the one launch — is emulated by an all-gather of the slices at launch time;
the run itself is the oracle's restatement of the reference driver
(oracle/bm_oracle.c: run_driver, gpu_match.cpp:306-376) on the assembled graph
and initial matching, and each rank keeps its own rows' and columns' slices of
the result.
"""
from __future__ import annotations

import pickle

import numpy as np


class CpuRank:
    def __init__(self, rank: int, world: int, transport):
        self.rank, self.world, self.x = rank, world, transport
        self.blob_bytes = 0

    def close(self):
        pass

    def upload(self, g, cb, rb):
        lo, hi = cb[self.rank], cb[self.rank + 1]
        base = int(g.cxadj[lo])
        self.cx = (g.cxadj[lo:hi + 1] - base).astype(np.int64)
        self.adj = np.asarray(g.cadj[base:int(g.cxadj[hi])], np.int32)
        self.nc, self.nr, self.cb, self.rb = g.nc, g.nr, list(cb), list(rb)
        self.row_index = False

    def export(self) -> bytes:
        return pickle.dumps((self.rank, self.cx, self.adj))

    def import_(self, blobs):
        parts = sorted((pickle.loads(b) for b in blobs), key=lambda t: t[0])
        assert [p[0] for p in parts] == list(range(self.world)), "blobs must come from every rank"
        cx = [np.zeros(1, np.int64)]
        adj = []
        off = 0
        for _, c, a in parts:
            cx.append(c[1:] + off)
            adj.append(a)
            off += int(c[-1])
        from paper_1303_1379_b200.api import BipartiteCsr
        self.g = BipartiteCsr(self.nc, self.nr, np.concatenate(cx), np.concatenate(adj) if adj else
                              np.zeros(0, np.int32), "assembled")

    def row_index_begin(self):
        self.row_index = "begun"

    def row_index_end(self):
        assert self.row_index == "begun", "row_index_end before row_index_begin"
        self.row_index = True

    def load(self, m):
        self.r0 = np.asarray(m.rmatch[self.rb[self.rank]:self.rb[self.rank + 1]], np.int32).copy()
        self.c0 = np.asarray(m.cmatch[self.cb[self.rank]:self.cb[self.rank + 1]], np.int32).copy()

    def launch(self, opts):
        from oracle import Oracle
        parts = self.x.allgather_obj((self.rank, self.r0.tobytes(), self.c0.tobytes()))
        rm = np.empty(self.nr, np.int32)
        cm = np.empty(self.nc, np.int32)
        for q, rb_, cb_ in parts:
            rm[self.rb[q]:self.rb[q + 1]] = np.frombuffer(rb_, np.int32)
            cm[self.cb[q]:self.cb[q + 1]] = np.frombuffer(cb_, np.int32)
        st, r, c, ct = Oracle().driver(self.g, rm, cm, shortest=bool(opts.driver), kernel=int(opts.bfs_kernel),
                                       improved=bool(opts.improved))
        assert st == 0, f"oracle driver status {st}"
        self.res = (r, c, ct)

    def finish(self):
        from paper_1303_1379_b200._lib import bm_counters
        r, c, ct = self.res
        out = bm_counters()
        out.outer_iterations = int(ct.get("outer_iterations", 0)) if isinstance(ct, dict) else 0
        out.cardinality = int((r >= 0).sum())
        return out.cardinality, out

    def download(self):
        r, c, _ = self.res
        return (r[self.rb[self.rank]:self.rb[self.rank + 1]].copy(), c[self.cb[self.rank]:self.cb[self.rank + 1]].copy())

    def kernel_ms(self) -> float:
        return 0.0
