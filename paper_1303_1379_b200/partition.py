"""1-D column-partitioned matching over several GPUs.

One process per GPU. Rank p owns the columns [p*nc//P, (p+1)*nc//P) with their
CSC slice; rmatch / cmatch / pred are replicated. A phase of APFB/APsB
(gpu_match.cpp:268-302, 306-376) becomes

    begin_phase                 every rank: its unmatched columns are roots
    repeat (one BFS level, gpubfs / gpubfs_wr, gpu_match.cpp:23-135):
        expand                  every rank: its frontier -> claim / endpoint records
        all-gather              records of all ranks, rank-major (NCCL over NVLink)
        merge                   every rank applies ALL records in the same order:
                                lowest (rank, index) wins per column and per free row,
                                so the replicas stay identical without further traffic
    end_bfs                     every rank: clear the visited bits
    augment                     rank 0: ALTERNATE + FIX (gpu_match.cpp:144-245)
    broadcast rmatch, cmatch    from rank 0

The all-gather is the only data-path exchange per level; the merge result
(next-frontier size, path found) is identical on every rank, so no extra
all-reduce is needed. The device side is the C ABI bm_part_* (bm_partition.cu);
``Exchange`` moves the records (torch.distributed: NCCL on device tensors, or
gloo with host staging), and the backend is pluggable so the protocol can be
exercised on CPU with gloo in the tests.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib
from .api import BfsKernel, BipartiteCsr, MatchingState

_vp = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)

_PART_PROTOS = {
    "bm_part_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "bm_part_destroy": (C.c_int, [_vp]),
    "bm_part_set_stream": (C.c_int, [_vp, _vp]),
    "bm_part_upload": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _i64p, _i32p]),
    "bm_part_bind_state": (C.c_int, [_vp, _vp, _vp]),
    "bm_part_record_capacity": (C.c_int, [_vp, _i64p, _i64p]),
    "bm_part_begin_phase": (C.c_int, [_vp, C.c_int32, C.c_int32, _i64p]),
    "bm_part_expand": (C.c_int, [_vp, _vp, _vp, _i32p, _i32p]),
    "bm_part_merge": (C.c_int, [_vp, _vp, _i32p, C.c_int64, _vp, _i32p, C.c_int64, _i64p, _i32p]),
    "bm_part_end_bfs": (C.c_int, [_vp]),
    "bm_part_augment": (C.c_int, [_vp, C.c_int32, _i64p]),
    "bm_part_cardinality": (C.c_int, [_vp, _i64p]),
    "bm_part_stats": (C.c_int, [_vp, _i64p, _i64p, _i64p, _i64p, _i64p]),
    "bm_part_reset_stats": (C.c_int, [_vp]),
    "bm_part_launch_count": (C.c_int, [_vp, _i64p]),
    "bm_part_p2p_export": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp]),
    "bm_part_p2p_import": (C.c_int, [_vp, _vp]),
    "bm_part_expand_p2p": (C.c_int, [_vp, C.c_int32]),
    "bm_part_merge_p2p": (C.c_int, [_vp, C.c_int32, C.c_uint32, _i64p, _i32p]),
}
for _name, (_res, _args) in _PART_PROTOS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def column_range(nc: int, rank: int, world: int) -> tuple[int, int]:
    """Columns owned by `rank`: an even 1-D split."""
    return nc * rank // world, nc * (rank + 1) // world


def slice_csc(g: BipartiteCsr, lo: int, hi: int) -> tuple[np.ndarray, np.ndarray]:
    """CSC slice of columns [lo, hi): offsets rebased to 0, and their rows."""
    cx = g.cxadj[lo:hi + 1]
    base = int(cx[0])
    return (cx - base).astype(np.int64), g.cadj[base:int(cx[-1])]


class Exchange:
    """Moves records between ranks with torch.distributed. With NCCL the
    tensors stay on the device (all_gather_into_tensor over NVLink); with
    gloo they are staged through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def allgather_counts(self, counts):
        import torch
        dev = "cuda" if self.nccl else "cpu"
        t = torch.tensor(counts, dtype=torch.int64, device=dev)
        out = torch.empty(self.world * len(counts), dtype=torch.int64, device=dev)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy().reshape(self.world, len(counts))

    def allgather_records(self, local, stride: int):
        """local: int32 tensor (stride, 4) padded; returns (world*stride, 4) on local's device."""
        import torch
        if self.nccl:
            out = torch.empty((self.world * stride, 4), dtype=torch.int32, device=local.device)
            self.dist.all_gather_into_tensor(out, local.contiguous(), group=self.group)
            return out
        host = local.cpu()
        parts = [torch.empty_like(host) for _ in range(self.world)]
        self.dist.all_gather(parts, host, group=self.group)
        return torch.cat(parts).to(local.device)

    def barrier(self):
        self.dist.barrier(group=self.group)

    def allgather_bytes(self, data: bytes) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, data, group=self.group)
        return out

    def broadcast_(self, t, src: int = 0):
        if self.nccl or t.device.type == "cpu":
            self.dist.broadcast(t, src, group=self.group)
            return t
        host = t.cpu()
        self.dist.broadcast(host, src, group=self.group)
        t.copy_(host)
        return t


class GpuPartition:
    """Device backend: one bm_part (this rank's slice on its GPU)."""

    def __init__(self, device: int, rank: int, world: int):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.rank, self.world = rank, world
        h = _vp()
        check(lib.bm_part_create(device, rank, world, C.byref(h)))
        self._h = h
        self.rmatch = self.cmatch = None
        # run on torch's current stream so the exchange and the kernels are ordered
        self.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def close(self):
        if getattr(self, "_h", None):
            lib.bm_part_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, ptr):
        check(lib.bm_part_set_stream(self._h, _vp(ptr)))

    def upload(self, nc: int, nr: int, lo: int, hi: int, cxs: np.ndarray, adjs: np.ndarray):
        torch = self.torch
        cxs = np.ascontiguousarray(cxs, dtype=np.int64)
        adjs = np.ascontiguousarray(adjs, dtype=np.int32)
        check(lib.bm_part_upload(self._h, nc, nr, lo, hi, cxs.ctypes.data_as(_i64p), adjs.ctypes.data_as(_i32p)))
        self.nc, self.nr = nc, nr
        self.rmatch = torch.empty(max(nr, 1), dtype=torch.int32, device=self.device)
        self.cmatch = torch.empty(max(nc, 1), dtype=torch.int32, device=self.device)
        check(lib.bm_part_bind_state(self._h, _vp(self.rmatch.data_ptr()), _vp(self.cmatch.data_ptr())))
        cc, ce = C.c_int64(), C.c_int64()
        check(lib.bm_part_record_capacity(self._h, C.byref(cc), C.byref(ce)))
        self.claims = torch.empty((cc.value, 4), dtype=torch.int32, device=self.device)
        self.eps = torch.empty((ce.value, 4), dtype=torch.int32, device=self.device)

    def load(self, m: MatchingState):
        torch = self.torch
        self.rmatch[:self.nr].copy_(torch.from_numpy(np.ascontiguousarray(m.rmatch, dtype=np.int32)))
        self.cmatch[:self.nc].copy_(torch.from_numpy(np.ascontiguousarray(m.cmatch, dtype=np.int32)))
        self.torch.cuda.synchronize(self.device)

    def begin_phase(self, kernel: int, endpoint_policy: int) -> int:
        n = C.c_int64()
        check(lib.bm_part_begin_phase(self._h, kernel, endpoint_policy, C.byref(n)))
        return n.value

    def expand(self):
        a, b = C.c_int32(), C.c_int32()
        self.torch.cuda.current_stream(self.device).synchronize()
        check(lib.bm_part_expand(self._h, _vp(self.claims.data_ptr()), _vp(self.eps.data_ptr()), C.byref(a), C.byref(b)))
        return self.claims, self.eps, a.value, b.value

    def merge(self, claims_all, claim_counts, cstride, eps_all, ep_counts, estride):
        self.torch.cuda.current_stream(self.device).synchronize()
        cc = np.ascontiguousarray(claim_counts, dtype=np.int32)
        ec = np.ascontiguousarray(ep_counts, dtype=np.int32)
        nxt, found = C.c_int64(), C.c_int32()
        check(lib.bm_part_merge(self._h, _vp(claims_all.data_ptr()), cc.ctypes.data_as(_i32p), cstride,
                                _vp(eps_all.data_ptr()), ec.ctypes.data_as(_i32p), estride,
                                C.byref(nxt), C.byref(found)))
        return nxt.value, bool(found.value)

    # -- fused P2P exchange (peer memory over NVLink, CUDA IPC)
    def p2p_export(self, claims_cap: int, endpoints_cap: int) -> bytes:
        buf = C.create_string_buffer(4 * 64)
        check(lib.bm_part_p2p_export(self._h, claims_cap, endpoints_cap, C.cast(buf, _vp)))
        return buf.raw

    def p2p_import(self, handles: bytes):
        buf = C.create_string_buffer(handles, len(handles))
        check(lib.bm_part_p2p_import(self._h, C.cast(buf, _vp)))

    def expand_p2p(self, parity: int):
        self.torch.cuda.current_stream(self.device).synchronize()
        check(lib.bm_part_expand_p2p(self._h, parity))

    def merge_p2p(self, parity: int, arrivals: int):
        nxt, found = C.c_int64(), C.c_int32()
        check(lib.bm_part_merge_p2p(self._h, parity, arrivals & 0xFFFFFFFF, C.byref(nxt), C.byref(found)))
        return nxt.value, bool(found.value)

    def end_bfs(self):
        check(lib.bm_part_end_bfs(self._h))

    def augment(self, serial: bool) -> int:
        card = C.c_int64()
        check(lib.bm_part_augment(self._h, 1 if serial else 0, C.byref(card)))
        return card.value

    def cardinality(self) -> int:
        self.torch.cuda.current_stream(self.device).synchronize()
        card = C.c_int64()
        check(lib.bm_part_cardinality(self._h, C.byref(card)))
        return card.value

    def state(self):
        return self.rmatch, self.cmatch

    def stats(self) -> dict:
        v = [C.c_int64() for _ in range(5)]
        check(lib.bm_part_stats(self._h, *[C.byref(x) for x in v]))
        keys = ["edges_traversed", "columns_scanned", "walks", "walk_steps", "fix_resets"]
        out = {k: x.value for k, x in zip(keys, v)}
        n = C.c_int64()
        check(lib.bm_part_launch_count(self._h, C.byref(n)))
        out["launches"] = n.value
        return out

    def reset_stats(self):
        check(lib.bm_part_reset_stats(self._h))

    def download(self) -> MatchingState:
        self.torch.cuda.synchronize(self.device)
        return MatchingState(self.rmatch[:self.nr].cpu().numpy().copy(), self.cmatch[:self.nc].cpu().numpy().copy())


@dataclass
class PartitionResult:
    cardinality: int
    phases: int
    levels: int
    serial_retries: int
    launches_per_phase: list = field(default_factory=list)
    records_exchanged: int = 0
    stats: dict = field(default_factory=dict)


class PartitionedMatcher:
    """The host loop of the partitioned driver (run_driver, gpu_match.cpp:306-359)."""

    def __init__(self, backend, exchange: Exchange):
        import os
        self.b = backend
        self.x = exchange
        self.rank, self.world = exchange.rank, exchange.world
        self.timing = os.environ.get("BM_PART_TIMING") == "1"  # host wall time per stage (profiling)
        self.t = {}

    def _tick(self, key, t0):
        import time
        if self.timing:
            t1 = time.perf_counter()
            self.t[key] = self.t.get(key, 0.0) + (t1 - t0)
            return t1
        return t0

    def upload(self, g: BipartiteCsr, p2p: bool = False):
        """Uploads this rank's slice. p2p: set up the fused exchange (records written
        straight into every rank's receive slabs over peer memory) instead of the
        all-gather through torch.distributed."""
        lo, hi = column_range(g.nc, self.rank, self.world)
        cxs, adjs = slice_csc(g, lo, hi)
        self.b.upload(g.nc, g.nr, lo, hi, cxs, adjs)
        self.nc, self.nr = g.nc, g.nr
        self.p2p = False
        if p2p:
            max_e = max(int(g.cxadj[column_range(g.nc, r, self.world)[1]] - g.cxadj[column_range(g.nc, r, self.world)[0]])
                        for r in range(self.world))
            self.x.barrier()  # no rank still maps a slab about to be replaced
            h = self.b.p2p_export(max(1, min(g.nc, max_e)), max(1, min(g.nr, max_e)))
            allh = self.x.allgather_bytes(h)
            self.b.p2p_import(b"".join(allh))
            self.p2p = True
            self.arrivals = 0

    def _gather(self, local, n_local: int, counts):
        """All-gather this rank's records, padded to the largest count."""
        stride = max(int(counts.max()), 1)
        if local.shape[0] >= stride:
            buf = local[:stride]
        else:  # another rank holds more records than this rank's buffer can
            import torch
            buf = torch.zeros((stride, 4), dtype=local.dtype, device=local.device)
            buf[:n_local] = local[:n_local]
        return self.x.allgather_records(buf, stride), stride

    def match(self, init: MatchingState, *, shortest: bool = False, kernel=BfsKernel.GpubfsWr,
              endpoint_policy: int = 0) -> PartitionResult:
        b = self.b
        b.load(init)
        b.reset_stats()
        before = b.cardinality()
        res = PartitionResult(cardinality=before, phases=0, levels=0, serial_retries=0)
        bound = self.nc + 1
        serial = False
        while True:
            res.phases += 1
            if res.phases > bound:
                raise RuntimeError("termination bound exceeded: more than nc + 1 phases")
            import time
            t0 = time.perf_counter()
            b.begin_phase(int(kernel), endpoint_policy)
            t0 = self._tick("begin", t0)
            found = False
            levels = 0
            while True:
                if self.p2p:  # fused exchange: no collective call, arrivals counted on the device
                    parity = (self.arrivals // self.world) & 1  # alternates every level, across phases too
                    b.expand_p2p(parity)
                    t0 = self._tick("expand", t0)
                    self.arrivals += self.world
                    n_next, found = b.merge_p2p(parity, self.arrivals)
                    t0 = self._tick("merge", t0)
                else:
                    claims, eps, nc_l, ne_l = b.expand()
                    t0 = self._tick("expand", t0)
                    counts = self.x.allgather_counts([nc_l, ne_l])
                    t0 = self._tick("counts", t0)
                    call, cstride = self._gather(claims, nc_l, counts[:, 0])
                    eall, estride = self._gather(eps, ne_l, counts[:, 1])
                    t0 = self._tick("gather", t0)
                    res.records_exchanged += int(counts.sum())
                    n_next, found = b.merge(call, counts[:, 0], cstride, eall, counts[:, 1], estride)
                    t0 = self._tick("merge", t0)
                levels += 1
                if (shortest and found) or n_next == 0:
                    break
            b.end_bfs()
            if self.rank == 0:
                b.augment(serial)
            t0 = self._tick("augment", t0)
            rm, cm = b.state()
            self.x.broadcast_(rm, 0)
            self.x.broadcast_(cm, 0)
            after = b.cardinality()
            t0 = self._tick("broadcast", t0)
            res.levels += levels
            res.launches_per_phase.append(levels)
            if found and after <= before and not serial:
                # a raced phase found a path but realised none (gpu_match.cpp:328-343):
                # redo it with a single-thread ALTERNATE on rank 0
                serial = True
                res.serial_retries += 1
                res.phases -= 1  # the retry belongs to the same outer iteration
                continue
            serial = False
            before = after
            if not found:
                break
        res.cardinality = before
        res.stats = b.stats()
        return res
