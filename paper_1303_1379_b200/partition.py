"""Multi-GPU matching over a 1-D column partition.

The device side is the multi-GPU engine (csrc/bm_mg.cu, C ABI ``bm_mg_*``):
the same persistent driver kernel as one GPU, one cooperative launch per
rank for the whole APFB/APsB run (run_driver, gpu_match.cpp:306-376). Rank q
owns the columns ``[cb[q], cb[q+1])`` with their CSC slice and the rows
``[rb[q], rb[q+1])`` with their row state; other ranks' state is reached over
peer memory (claims are system-scope atomics at the row's owner, winner
columns go straight into their owner's inbox, the level barrier spans the
team). This module is the host protocol around it:

    upload      every rank: its column slice (bm_mg_partition bounds)
    exchange    every rank's peer-pointer blob -> all ranks (all-gather)
    row index   (pulled levels) bucket own edges; barrier; gather own rows
    load        every rank: the initial matching of its rows and columns
    run         every rank launches, then waits (one launch per run)
    download    every rank: its rows and columns; gathered on demand

Two transports carry the setup messages (never the data path):
``LocalTransport`` for several ranks in one process (each on its own CUDA
stream, e.g. sharing one GPU in tests), and ``DistTransport``
(torch.distributed, one process per GPU, NCCL or gloo). The backend is
pluggable so that the protocol runs on CPU with the oracle standing in for the
device (``oracle.partition_ref``) in the gloo tests.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import bm_counters, bm_match_opts, check, lib
from .api import BfsKernel, BipartiteCsr, MatchingState, _bu_mode, _opts

_vp = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)

_MG_PROTOS = {
    "bm_mg_partition": (C.c_int, [C.c_int32, C.c_int32, _i32p]),
    "bm_mg_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "bm_mg_destroy": (C.c_int, [_vp]),
    "bm_mg_set_stream": (C.c_int, [_vp, _vp]),
    "bm_mg_upload": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int64, _i32p, _i32p, _i64p, _i32p]),
    "bm_mg_blob_size": (C.c_int, [_i64p]),
    "bm_mg_export": (C.c_int, [_vp, _vp]),
    "bm_mg_import": (C.c_int, [_vp, _vp]),
    "bm_mg_row_index_begin": (C.c_int, [_vp]),
    "bm_mg_row_index_end": (C.c_int, [_vp]),
    "bm_mg_load_matching": (C.c_int, [_vp, _i32p, _i32p]),
    "bm_mg_launch": (C.c_int, [_vp, C.POINTER(bm_match_opts)]),
    "bm_mg_finish": (C.c_int, [_vp, _i64p, C.POINTER(bm_counters)]),
    "bm_mg_download": (C.c_int, [_vp, _i32p, _i32p]),
    "bm_mg_kernel_time": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "bm_mg_info": (C.c_int, [_vp, _i64p, _i64p, _i32p]),
}
for _name, (_res, _args) in _MG_PROTOS.items():
    if hasattr(lib, _name):
        _fn = getattr(lib, _name)
        _fn.restype = _res
        _fn.argtypes = _args


def partition_bounds(n: int, world: int) -> list:
    """The engine's split of n ids over world ranks: even, inner bounds 32-aligned."""
    b = (C.c_int32 * (world + 1))()
    check(lib.bm_mg_partition(n, world, b))
    return list(b)


def column_range(nc: int, rank: int, world: int) -> tuple:
    """Columns owned by `rank` (bm_mg_partition)."""
    b = partition_bounds(nc, world)
    return b[rank], b[rank + 1]


def slice_csc(g: BipartiteCsr, lo: int, hi: int) -> tuple:
    """CSC slice of columns [lo, hi): offsets rebased to 0, and their rows."""
    cx = g.cxadj[lo:hi + 1]
    base = int(cx[0])
    return (cx - base).astype(np.int64), g.cadj[base:int(cx[-1])]


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class GpuRank:
    """One rank of the multi-GPU engine (a bm_mg handle)."""

    def __init__(self, device: int, rank: int, world: int, share: int = 1):
        h = _vp()
        check(lib.bm_mg_create(device, rank, world, share, C.byref(h)))
        self._h = h
        self.device, self.rank, self.world = device, rank, world
        n = C.c_int64()
        check(lib.bm_mg_blob_size(C.byref(n)))
        self.blob_bytes = n.value

    def close(self):
        if getattr(self, "_h", None):
            lib.bm_mg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, ptr):
        check(lib.bm_mg_set_stream(self._h, _vp(ptr)))

    def upload(self, g: BipartiteCsr, cb: list, rb: list, slices=None):
        """This rank's column slice of g (or the given (cxadj, cadj) slice,
        e.g. in pinned host memory)."""
        lo, hi = cb[self.rank], cb[self.rank + 1]
        cx, adj = slices if slices is not None else slice_csc(g, lo, hi)
        cx = np.ascontiguousarray(cx, np.int64)
        adj = np.ascontiguousarray(adj, np.int32)
        cba = np.asarray(cb, np.int32)
        rba = np.asarray(rb, np.int32)
        check(lib.bm_mg_upload(self._h, g.nc, g.nr, g.num_edges(), _ptr(cba, C.c_int32), _ptr(rba, C.c_int32),
                               _ptr(cx, C.c_int64), _ptr(adj, C.c_int32)))
        self.cb, self.rb = list(cb), list(rb)

    def export(self) -> bytes:
        buf = C.create_string_buffer(self.blob_bytes)
        check(lib.bm_mg_export(self._h, C.cast(buf, _vp)))
        return buf.raw

    def import_(self, blobs: list):
        raw = b"".join(blobs)
        buf = C.create_string_buffer(raw, len(raw))
        check(lib.bm_mg_import(self._h, C.cast(buf, _vp)))

    def row_index_begin(self):
        check(lib.bm_mg_row_index_begin(self._h))

    def row_index_end(self):
        check(lib.bm_mg_row_index_end(self._h))

    def load(self, m: MatchingState, slices=None):
        """The initial matching of this rank's rows and columns (taken from the whole
        arrays of m, or given directly as `slices` = (rows, cols), e.g. pinned)."""
        if slices is not None:
            r, c = slices
        else:
            r = np.ascontiguousarray(m.rmatch[self.rb[self.rank]:self.rb[self.rank + 1]], np.int32)
            c = np.ascontiguousarray(m.cmatch[self.cb[self.rank]:self.cb[self.rank + 1]], np.int32)
        check(lib.bm_mg_load_matching(self._h, _ptr(r, C.c_int32), _ptr(c, C.c_int32)))

    def launch(self, opts: bm_match_opts):
        check(lib.bm_mg_launch(self._h, C.byref(opts)))

    def finish(self):
        card = C.c_int64()
        ct = bm_counters()
        check(lib.bm_mg_finish(self._h, C.byref(card), C.byref(ct)))
        return card.value, ct

    def download(self, out=None):
        """This rank's rows and columns; `out` = (rows, cols) caller arrays (e.g. pinned)."""
        if out is None:
            out = (np.empty(self.rb[self.rank + 1] - self.rb[self.rank], np.int32),
                   np.empty(self.cb[self.rank + 1] - self.cb[self.rank], np.int32))
        r, c = out
        check(lib.bm_mg_download(self._h, _ptr(r, C.c_int32), _ptr(c, C.c_int32)))
        return r, c

    def kernel_ms(self) -> float:
        ms = C.c_double()
        check(lib.bm_mg_kernel_time(self._h, C.byref(ms)))
        return ms.value

    def info(self) -> dict:
        a, b, c = C.c_int64(), C.c_int64(), C.c_int32()
        check(lib.bm_mg_info(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"local_edges": a.value, "row_index_edges": b.value, "pulled_capable": bool(c.value)}


class LocalTransport:
    """Setup messages between ranks that live in this process."""

    def allgather(self, items: list) -> list:
        return list(items)

    def barrier(self):
        pass


class DistTransport:
    """Setup messages over torch.distributed (one rank per process)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def allgather_obj(self, obj):
        out = [None] * self.dist.get_world_size(self.group)
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier(self):
        self.dist.barrier(group=self.group)

    def allreduce_max(self, x: float) -> float:
        out = self.allgather_obj(float(x))
        return max(out)

    def allreduce_sum(self, x: int) -> int:
        return sum(self.allgather_obj(int(x)))


@dataclass
class TeamResult:
    cardinality: int
    phases: int
    levels: int
    serial_retries: int
    kernel_ms: float
    counters: list = field(default_factory=list)  # per local rank
    launches_per_phase: list = field(default_factory=list)


def _opts_for(shortest, kernel, improved, bottom_up, init_mode="given"):
    o = _opts(shortest, kernel, improved, init_mode)
    o.bottom_up = _bu_mode(bottom_up)
    return o


class LocalTeam:
    """All ranks of the team in this process (one stream each). With every
    rank on one GPU this exercises the whole protocol and the kernels' peer
    addressing on a single device."""

    def __init__(self, world: int, devices=None):
        import torch
        self.world = world
        devices = list(devices) if devices is not None else [0] * world
        share = {d: devices.count(d) for d in devices}
        self.ranks = [GpuRank(devices[q], q, world, share[devices[q]]) for q in range(world)]
        self.streams = []
        for q, r in enumerate(self.ranks):
            s = torch.cuda.Stream(device=devices[q])
            self.streams.append(s)
            r.set_stream(s.cuda_stream)
        self.g = None

    def close(self):
        for r in self.ranks:
            r.close()

    def upload(self, g: BipartiteCsr, row_index: bool = False):
        cb = partition_bounds(g.nc, self.world)
        rb = partition_bounds(g.nr, self.world)
        for r in self.ranks:
            r.upload(g, cb, rb)
        blobs = [r.export() for r in self.ranks]
        for r in self.ranks:
            r.import_(blobs)
        if row_index:
            for r in self.ranks:
                r.row_index_begin()
            for r in self.ranks:
                r.row_index_end()
        self.g, self.cb, self.rb = g, cb, rb

    def match(self, init: MatchingState, *, shortest=False, kernel=BfsKernel.GpubfsWr, improved=False,
              bottom_up="auto", init_mode="given") -> tuple:
        opts = _opts_for(shortest, kernel, improved, bottom_up, init_mode)
        for r in self.ranks:
            r.load(init)
        for r in self.ranks:
            r.launch(opts)
        outs = [r.finish() for r in self.ranks]
        cards = {c for c, _ in outs}
        assert len(cards) == 1, f"ranks disagree on the cardinality: {cards}"
        ct = outs[0][1]
        res = TeamResult(cardinality=outs[0][0], phases=ct.outer_iterations, levels=ct.bfs_launches_total,
                         serial_retries=ct.serial_retries, kernel_ms=max(r.kernel_ms() for r in self.ranks),
                         counters=[c for _, c in outs])
        return res, self.gather()

    def gather(self) -> MatchingState:
        g = self.g
        rm = np.empty(g.nr, np.int32)
        cm = np.empty(g.nc, np.int32)
        for r in self.ranks:
            a, b = r.download()
            rm[self.rb[r.rank]:self.rb[r.rank + 1]] = a
            cm[self.cb[r.rank]:self.cb[r.rank + 1]] = b
        return MatchingState(rm, cm)


class PartitionedMatcher:
    """One rank of a team spread over processes (torch.distributed, one GPU
    each). ``backend`` is a GpuRank, or the oracle stand-in on CPU."""

    def __init__(self, backend, transport: DistTransport):
        self.b = backend
        self.x = transport
        self.rank, self.world = backend.rank, backend.world

    def upload(self, g: BipartiteCsr, row_index: bool = False, slices=None):
        cb = partition_bounds(g.nc, self.world)
        rb = partition_bounds(g.nr, self.world)
        if slices is not None:
            self.b.upload(g, cb, rb, slices)
        else:
            self.b.upload(g, cb, rb)
        blobs = self.x.allgather_obj(self.b.export())
        self.b.import_(blobs)
        if row_index:
            self.b.row_index_begin()
            self.x.barrier()  # every outbox is complete before anyone gathers from it
            self.b.row_index_end()
        self.x.barrier()
        self.g, self.cb, self.rb = g, cb, rb

    def match(self, init: MatchingState, *, shortest=False, kernel=BfsKernel.GpubfsWr, improved=False,
              bottom_up="auto", init_mode="given", slices=None) -> TeamResult:
        opts = _opts_for(shortest, kernel, improved, bottom_up, init_mode)
        if slices is None:
            self.b.load(init)
        else:
            self.b.load(init, slices=slices)
        self.x.barrier()  # no kernel touches a peer's state before that peer loaded it
        self.b.launch(opts)
        card, ct = self.b.finish()
        return TeamResult(cardinality=card, phases=ct.outer_iterations, levels=ct.bfs_launches_total,
                          serial_retries=ct.serial_retries, kernel_ms=self.b.kernel_ms(), counters=[ct])

    def gather(self) -> MatchingState:
        """The whole matching on every rank (all-gather of the slices)."""
        rs, cs = self.b.download()
        parts = self.x.allgather_obj((self.rank, rs.tobytes(), cs.tobytes()))
        rm = np.empty(self.g.nr, np.int32)
        cm = np.empty(self.g.nc, np.int32)
        for q, rb_, cb_ in parts:
            rm[self.rb[q]:self.rb[q + 1]] = np.frombuffer(rb_, np.int32)
            cm[self.cb[q]:self.cb[q + 1]] = np.frombuffer(cb_, np.int32)
        return MatchingState(rm, cm)
