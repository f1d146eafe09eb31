"""Python mirror of the reference's public interface for the matching hot path.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj), so code written against it reads the same here:

  BipartiteCsr, check_csr                 include/bmatch/csr_graph.hpp:18-49
  MatchingState, cheap_matching,
  cardinality                             include/bmatch/matching.hpp:15-33
  BfsKernel, PhaseCounters, PhaseEvent,
  DriverResult, apfb, apsb                include/bmatch/gpu_match.hpp:13-144
  AlgorithmResult, algorithm_ids,
  make_algorithm, register_algorithm      include/bmatch/algorithms.hpp:15-42
  ParseError, read_matrix_market,
  load_matrix_market, write_matrix_market include/bmatch/matrix_market.hpp:10-24

Every matching call goes through the C ABI (libbmatch_b200.so) to the sm_100a
engine; `grid` and `schedule` are accepted for signature compatibility and
ignored (the device sizes its own grid). The C++ drop-in for the reference's
own registry is include/bmatch_b200.hpp.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._lib import CudaError, LogicError, ParseError, check, i32p, i64p, lib

__all__ = [
    "BfsKernel", "BipartiteCsr", "MatchingState", "PhaseCounters", "PhaseEvent", "DriverResult",
    "AlgorithmResult", "Engine", "apfb", "apsb", "cheap_matching", "cardinality", "check_csr",
    "csc_digest", "algorithm_ids", "make_algorithm", "register_algorithm", "generate_random_bipartite",
    "generate_planted", "generate_rmat", "generate_banded", "LogicError", "CudaError", "INIT_MODES",
    "permutation_pair", "ParseError", "read_matrix_market", "load_matrix_market", "write_matrix_market",
    "save_csc", "load_csc",
]

INIT_MODES = {"given": _lib.BM_INIT_GIVEN, "gpu_greedy": _lib.BM_INIT_GPU_GREEDY, "gpu_ks": _lib.BM_INIT_GPU_KS}


class BfsKernel(enum.IntEnum):
    """gpu_match.hpp:13"""
    Gpubfs = 0
    GpubfsWr = 1


@dataclass
class BipartiteCsr:
    """CSC graph: rows of column c are cadj[cxadj[c]:cxadj[c+1]] (csr_graph.hpp:18-31)."""
    nc: int
    nr: int
    cxadj: np.ndarray  # int64[nc+1]
    cadj: np.ndarray   # int32[E]
    name: str = ""

    def __post_init__(self):
        self.cxadj = np.ascontiguousarray(self.cxadj, dtype=np.int64)
        self.cadj = np.ascontiguousarray(self.cadj, dtype=np.int32)

    def num_edges(self) -> int:
        return int(self.cxadj[-1]) if len(self.cxadj) else 0

    def column(self, c: int) -> np.ndarray:
        return self.cadj[self.cxadj[c]:self.cxadj[c + 1]]

    @staticmethod
    def from_edge_list(nc: int, nr: int, edges, name: str = "") -> "BipartiteCsr":
        """csr_graph.cpp:10-43: sort, de-duplicate, out_of_range on bad ids."""
        e = np.asarray(list(edges), dtype=np.int64).reshape(-1, 2)
        for k, (c, r) in enumerate(e):
            if c < 0 or c >= nc:
                raise IndexError(f"edge {k} (c={c}, r={r}): column index outside [0, {nc})")
            if r < 0 or r >= nr:
                raise IndexError(f"edge {k} (c={c}, r={r}): row index outside [0, {nr})")
        if len(e):
            e = np.unique(e, axis=0)
        counts = np.bincount(e[:, 0], minlength=nc) if len(e) else np.zeros(nc, dtype=np.int64)
        cx = np.zeros(nc + 1, dtype=np.int64)
        cx[1:] = np.cumsum(counts)
        return BipartiteCsr(nc, nr, cx, e[:, 1].astype(np.int32) if len(e) else np.zeros(0, np.int32), name)


@dataclass
class MatchingState:
    """rmatch[r] in {-2,-1} U [0,nc); cmatch[c] in {-1} U [0,nr) (matching.hpp:15-25)."""
    rmatch: np.ndarray
    cmatch: np.ndarray

    def __post_init__(self):
        self.rmatch = np.ascontiguousarray(self.rmatch, dtype=np.int32)
        self.cmatch = np.ascontiguousarray(self.cmatch, dtype=np.int32)

    @staticmethod
    def unmatched(nc: int, nr: int) -> "MatchingState":
        return MatchingState(np.full(nr, -1, np.int32), np.full(nc, -1, np.int32))

    def copy(self) -> "MatchingState":
        return MatchingState(self.rmatch.copy(), self.cmatch.copy())


@dataclass
class PhaseCounters:
    """gpu_match.hpp:39-52, plus the device work counters used for the roofline."""
    outer_iterations: int = 0
    bfs_launches_per_iteration: list = field(default_factory=list)
    columns_scanned: int = 0
    alternations_attempted: int = 0
    fix_resets: int = 0
    serial_retries: int = 0
    edges_traversed: int = 0
    columns_visited: int = 0
    walk_steps: int = 0
    frontier_entries: int = 0
    initial_cardinality: int = 0

    def bfs_launches_total(self) -> int:
        return int(sum(self.bfs_launches_per_iteration))


@dataclass
class PhaseEvent:
    """gpu_match.hpp:115-123"""
    iteration: int
    augmenting_path_found: bool
    cardinality_before: int
    cardinality_after: int
    serial_retry: bool
    bfs_launches: int
    state: MatchingState


@dataclass
class DriverResult:
    matching: MatchingState
    counters: PhaseCounters


@dataclass
class AlgorithmResult:
    matching: MatchingState
    counters: Optional[PhaseCounters] = None


def _bu_mode(bottom_up) -> int:
    """bm_bottom_up from True / False / "auto" (or the int itself)."""
    if isinstance(bottom_up, str):
        return {"auto": _lib.BM_BU_AUTO, "on": _lib.BM_BU_ON, "off": _lib.BM_BU_OFF}[bottom_up]
    if isinstance(bottom_up, bool):
        return _lib.BM_BU_ON if bottom_up else _lib.BM_BU_OFF
    return int(bottom_up)


def _opts(shortest: bool, kernel: BfsKernel, improved: bool, init_mode: str, max_phases: int = 0,
          claim_mode: int = 0, endpoint_policy: int = 0, bottom_up="auto"):
    o = _lib.bm_match_opts()
    o.claim_policy = claim_mode
    o.endpoint_policy = endpoint_policy
    o.bottom_up = _bu_mode(bottom_up)
    o.driver = _lib.BM_DRIVER_APSB if shortest else _lib.BM_DRIVER_APFB
    o.bfs_kernel = int(kernel)
    o.improved = 1 if improved else 0
    if init_mode not in INIT_MODES:
        raise ValueError(f"unknown init mode {init_mode!r} (expected one of {sorted(INIT_MODES)})")
    o.init = INIT_MODES[init_mode]
    o.max_phases = max_phases
    return o


def _counters_from(ct: _lib.bm_counters, launches: np.ndarray) -> PhaseCounters:
    n = int(ct.n_phase_records)
    return PhaseCounters(
        outer_iterations=int(ct.outer_iterations),
        bfs_launches_per_iteration=[int(x) for x in launches[:n]],
        columns_scanned=int(ct.columns_scanned),
        alternations_attempted=int(ct.alternations_attempted),
        fix_resets=int(ct.fix_resets),
        serial_retries=int(ct.serial_retries),
        edges_traversed=int(ct.edges_traversed),
        columns_visited=int(ct.columns_visited),
        walk_steps=int(ct.walk_steps),
        frontier_entries=int(ct.frontier_entries),
        initial_cardinality=int(ct.initial_cardinality),
    )


class Engine:
    """One device handle (bm_handle): a device-resident CSC plus matching state.

    Not re-entrant; use one Engine per thread. Holds the last uploaded graph so
    repeated calls on the same BipartiteCsr object skip the H2D copy.
    """

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.bm_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self._graph = None
        self.bottom_up = "auto"  # bm_match_opts.bottom_up default for match()/run(): True, False or "auto"

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib.bm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        check(lib.bm_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    # -- graph
    def upload(self, g: BipartiteCsr, force: bool = False):
        if self._graph is g and not force:
            return
        self._graph = None
        check(lib.bm_upload_csc(self._h, g.nc, g.nr, i64p(g.cxadj), i32p(g.cadj)))
        self._graph = g

    def upload_ptrs(self, nc: int, nr: int, cxadj_ptr: int, cadj_ptr: int):
        """Upload from raw host pointers (e.g. pinned buffers)."""
        self._graph = None
        check(lib.bm_upload_csc(self._h, nc, nr, C.cast(C.c_void_p(cxadj_ptr), _lib._i64p),
                                C.cast(C.c_void_p(cadj_ptr), _lib._i32p)))

    # -- matching
    def match(self, g: BipartiteCsr, init: Optional[MatchingState], *, shortest=False,
              kernel=BfsKernel.GpubfsWr, improved=False, init_mode="given",
              observer: Optional[Callable[[PhaseEvent], None]] = None) -> DriverResult:
        m = init.copy() if init is not None else MatchingState.unmatched(g.nc, g.nr)
        ct, launches = self._match(g, m, shortest, kernel, improved, init_mode, observer)
        return DriverResult(m, _counters_from(ct, launches))

    def match_inplace(self, g: BipartiteCsr, m: MatchingState, *, shortest=False, kernel=BfsKernel.GpubfsWr,
                      improved=False, init_mode="given") -> int:
        """bm_match on caller-owned arrays (e.g. pinned buffers): m holds the
        initial matching on entry and the maximum matching on return."""
        ct, _ = self._match(g, m, shortest, kernel, improved, init_mode, None, want_launches=False)
        return int(ct.cardinality)

    def _match(self, g, m, shortest, kernel, improved, init_mode, observer, want_launches=True):
        self.upload(g)
        o = _opts(shortest, kernel, improved, init_mode, bottom_up=self.bottom_up)
        if len(m.rmatch) != g.nr or len(m.cmatch) != g.nc:
            raise ValueError("matching arrays do not fit the graph")
        ct = _lib.bm_counters()
        cap = g.nc + 2 if want_launches else 0
        launches = np.zeros(max(cap, 1), np.int64)
        card = C.c_int64()
        cb, err = self._make_cb(observer)
        st = lib.bm_match(self._h, C.byref(o), i32p(m.rmatch), i32p(m.cmatch), C.byref(card), C.byref(ct),
                          i64p(launches) if cap else None, cap, cb, None)
        if err:
            raise err[0]
        check(st)
        return ct, launches

    @staticmethod
    def _make_cb(observer):
        err: list = []
        if observer is None:
            return _lib.PHASE_CB(), err

        def _cb(ev_p, _user):
            ev = ev_p.contents
            try:
                state = MatchingState(np.ctypeslib.as_array(ev.rmatch, (ev.nr,)).copy() if ev.nr else
                                      np.zeros(0, np.int32),
                                      np.ctypeslib.as_array(ev.cmatch, (ev.nc,)).copy() if ev.nc else
                                      np.zeros(0, np.int32))
                observer(PhaseEvent(int(ev.iteration), bool(ev.augmenting_path_found),
                                    int(ev.cardinality_before), int(ev.cardinality_after),
                                    bool(ev.serial_retry), int(ev.bfs_launches), state))
                return 0
            except BaseException as e:  # surfaced after the C call returns
                err.append(e)
                return 1

        return _lib.PHASE_CB(_cb), err

    def load_matching(self, m: MatchingState):
        check(lib.bm_load_matching(self._h, i32p(m.rmatch), i32p(m.cmatch)))

    def run(self, *, shortest=False, kernel=BfsKernel.GpubfsWr, improved=False, init_mode="given",
            max_phases=0, observer=None, resume=False, claim_mode=0, endpoint_policy=0, bottom_up=None):
        """Device-resident run (bm_run / bm_resume). Returns (cardinality, counters, done).
        claim_mode / endpoint_policy: bm_claim_policy / bm_endpoint_policy (WR tuning knobs)."""
        o = _opts(shortest, kernel, improved, init_mode, max_phases, claim_mode, endpoint_policy,
                  self.bottom_up if bottom_up is None else bottom_up)
        ct = _lib.bm_counters()
        nc = self._nc()
        cap = nc + 2
        launches = np.zeros(cap, np.int64)
        card = C.c_int64()
        done = C.c_int32()
        cb, err = self._make_cb(observer)
        fn = lib.bm_resume if resume else lib.bm_run
        st = fn(self._h, C.byref(o), C.byref(card), C.byref(ct), i64p(launches), cap, cb, None, C.byref(done))
        if err:
            raise err[0]
        check(st)
        return int(card.value), _counters_from(ct, launches), bool(done.value)

    def download(self, nc: int | None = None, nr: int | None = None) -> MatchingState:
        gnc, gnr, _ = self.graph_info()
        m = MatchingState.unmatched(gnc, gnr)
        check(lib.bm_download_matching(self._h, i32p(m.rmatch), i32p(m.cmatch)))
        return m

    def bottom_up_auto(self) -> int:
        """BM_BU_AUTO for the resident graph (bmatch_b200.h): 0 pushes, 1 pulls dense
        levels once the row index is prepared, 2 pulls them from the first run."""
        v = C.c_int32()
        check(lib.bm_bottom_up_auto(self._h, C.byref(v)))
        return int(v.value)

    def prepare_row_index(self):
        """Build the row index now (bm_prepare_row_index), so "auto" pulls from the next run."""
        check(lib.bm_prepare_row_index(self._h))

    def last_phase_launches(self) -> list:
        """BFS launches per outer iteration of the last run (bm_last_phase_launches)."""
        n = C.c_int64()
        check(lib.bm_last_phase_launches(self._h, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.int64)
        check(lib.bm_last_phase_launches(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)), n.value, C.byref(n)))
        return [int(x) for x in out[:n.value]]

    def row_index(self):
        """The row index the pulled levels read (bm_download_row_index): (roffs[nr+1], radj[E])."""
        nc, nr, ne = self.graph_info()
        roffs = np.empty(nr + 1, np.uint32)
        radj = np.empty(max(ne, 1), np.int32)
        check(lib.bm_download_row_index(self._h, roffs.ctypes.data_as(C.POINTER(C.c_uint32)),
                                        radj.ctypes.data_as(C.POINTER(C.c_int32))))
        return roffs, radj[:ne]

    def graph_info(self):
        nc, nr, ne = C.c_int32(), C.c_int32(), C.c_int64()
        check(lib.bm_graph_info(self._h, C.byref(nc), C.byref(nr), C.byref(ne)))
        return nc.value, nr.value, ne.value

    def _nc(self) -> int:
        return self.graph_info()[0]

    DEBUG_PHASE_BOUND = 1
    DEBUG_SKIP_ALTERNATE_PHASE = 2

    def debug_set(self, key: int, value: int):
        """Fault injection for the failure-path tests (bm_debug_set)."""
        check(lib.bm_debug_set(self._h, key, value))

    def last_kernel_time(self):
        ms, n = C.c_double(), C.c_int32()
        check(lib.bm_last_kernel_time(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    TL_KINDS = {0: "start", 1: "init", 2: "setup", 3: "level", 4: "alternate", 5: "fix_rows", 6: "fix_cols",
                7: "roots", 8: "end", 9: "level_edges", 10: "materialize", 11: "pull_prep", 12: "bucketed",
                13: "late_level", 14: "late"}

    def timeline(self):
        """Stage timeline of the last run: list of (kind, arg, t_ns) from the device clock."""
        n = C.c_int64()
        check(lib.bm_timeline(self._h, None, 0, C.byref(n)))
        buf = np.zeros(2 * max(n.value, 1), np.uint64)
        check(lib.bm_timeline(self._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), n.value, C.byref(n)))
        out = []
        for i in range(n.value):
            tag, t = int(buf[2 * i]), int(buf[2 * i + 1])
            out.append((self.TL_KINDS.get(tag >> 32, str(tag >> 32)), tag & 0xFFFFFFFF, t))
        return out

    STAT_NAMES = ["edges_traversed", "columns_scanned", "columns_visited", "frontier_entries", "walks",
                  "walk_steps", "fix_resets", "levels", "serial_retries", "dense_fix", "cyc_tile", "cyc_window",
                  "cyc_rounds", "cyc_flush", "cyc_barrier", "cyc_other", "rows_pulled", "pulled_levels",
                  "materialized", "cyc_bu_screen", "cyc_bu_probe", "cyc_bu_flush", "bu_rounds",
                  "late_phases", "late_paths", "late_proofs"]

    def debug_stats(self) -> dict:
        buf = np.zeros(32, np.uint64)
        n = C.c_int64()
        check(lib.bm_debug_stats(self._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), 32, C.byref(n)))
        return {name: int(buf[i]) for i, name in enumerate(self.STAT_NAMES[:n.value])}

    def bfs_phase(self, g: BipartiteCsr, m: MatchingState, *, shortest=False, kernel=BfsKernel.Gpubfs,
                  improved=False):
        """One BFS expansion without ALTERNATE/FIX. Returns (bfs, pred, rmatch, launches, found)."""
        self.upload(g)
        bfs = np.zeros(g.nc, np.int32)
        pred = np.zeros(g.nr, np.int32)
        rm = np.zeros(g.nr, np.int32)
        launches, found = C.c_int64(), C.c_int32()
        check(lib.bm_bfs_phase(self._h, 1 if shortest else 0, int(kernel), 1 if improved else 0,
                               i32p(m.rmatch), i32p(m.cmatch), i32p(bfs), i32p(pred), i32p(rm),
                               C.byref(launches), C.byref(found)))
        return bfs, pred, rm, int(launches.value), bool(found.value)

    def permute_random(self, seed: int):
        """Relabel the resident graph on the device exactly as the reference's
        permute_random(g, seed) (csr_graph.cpp:80-90)."""
        gnc, gnr, _ = self.graph_info()
        cp, rp = permutation_pair(gnc, gnr, seed)
        check(lib.bm_permute_random(self._h, i32p(cp), i32p(rp)))
        self._graph = None

    def download_graph(self, name: str = "") -> BipartiteCsr:
        gnc, gnr, ne = self.graph_info()
        cx = np.zeros(gnc + 1, np.int64)
        adj = np.zeros(max(ne, 0), np.int32)
        check(lib.bm_download_csc(self._h, i64p(cx), i32p(adj)))
        return BipartiteCsr(gnc, gnr, cx, adj, name)

    def verify(self, g: BipartiteCsr, m: MatchingState):
        """GPU Berge certificate: (violations, is_maximum, cardinality)."""
        self.upload(g)
        v, ismax, card = C.c_int64(), C.c_int32(), C.c_int64()
        check(lib.bm_verify(self._h, i32p(m.rmatch), i32p(m.cmatch), C.byref(v), C.byref(ismax), C.byref(card)))
        return int(v.value), bool(ismax.value), int(card.value)


_tls = threading.local()


def default_engine(device: int = 0) -> Engine:
    engines = getattr(_tls, "engines", None)
    if engines is None:
        engines = _tls.engines = {}
    if device not in engines:
        engines[device] = Engine(device)
    return engines[device]


def apfb(g: BipartiteCsr, init: MatchingState, grid=None, schedule=None, kernel=BfsKernel.GpubfsWr,
         observer=None, *, init_mode="given", device=0) -> DriverResult:
    """Augment-all driver (gpu_match.hpp:131-135) on the B200 engine."""
    return default_engine(device).match(g, init, shortest=False, kernel=BfsKernel(kernel), improved=False,
                                        init_mode=init_mode, observer=observer)


def apsb(g: BipartiteCsr, init: MatchingState, grid=None, schedule=None, kernel=BfsKernel.GpubfsWr,
         improved_alternate=False, observer=None, *, init_mode="given", device=0) -> DriverResult:
    """Shortest-path driver (gpu_match.hpp:137-144) on the B200 engine."""
    if improved_alternate and BfsKernel(kernel) != BfsKernel.GpubfsWr:
        raise LogicError("the endpoint-encoded alternation requires the with-root kernel")
    return default_engine(device).match(g, init, shortest=True, kernel=BfsKernel(kernel),
                                        improved=improved_alternate, init_mode=init_mode, observer=observer)


def permutation_pair(nc: int, nr: int, seed: int):
    """(cperm, rperm) of the reference's permute_random(g, seed) (csr_graph.cpp:68-90)."""
    cp = np.zeros(max(nc, 0), np.int32)
    rp = np.zeros(max(nr, 0), np.int32)
    check(lib.bm_permutation_pair(nc, nr, seed, i32p(cp), i32p(rp)))
    return cp, rp


def cheap_matching(g: BipartiteCsr) -> MatchingState:
    """First-fit greedy in ascending column order (matching.cpp:13-26), host side."""
    m = MatchingState.unmatched(g.nc, g.nr)
    check(lib.bm_host_cheap_matching(g.nc, g.nr, i64p(g.cxadj), i32p(g.cadj), i32p(m.rmatch), i32p(m.cmatch)))
    return m


def cardinality(m: MatchingState) -> int:
    """matching.cpp:28-31"""
    return int(np.count_nonzero(m.rmatch >= 0))


def check_csr(g: BipartiteCsr) -> None:
    """csr_graph.cpp:45-64 (raises ValueError, the analogue of std::logic_error there)."""
    if len(g.cxadj) != g.nc + 1:
        raise ValueError("cxadj length is not nc + 1")
    if int(g.cxadj[-1]) != len(g.cadj):
        raise ValueError("cxadj[nc] does not match cadj length")
    check(lib.bm_check_csc(g.nc, g.nr, i64p(g.cxadj), i32p(g.cadj)))


def csc_digest(g: BipartiteCsr) -> int:
    return int(lib.bm_csc_digest(g.nc, g.nr, i64p(g.cxadj), i32p(g.cadj)))


# ---- registry (algorithms.hpp:15-42) ---------------------------------------
_GRID_ALGOS = {
    # id: (shortest, kernel, improved) — algorithms.cpp:19-27
    "apfb-gpubfs": (False, BfsKernel.Gpubfs, False),
    "apfb-wr": (False, BfsKernel.GpubfsWr, False),
    "apsb-gpubfs": (True, BfsKernel.Gpubfs, False),
    "apsb-wr": (True, BfsKernel.GpubfsWr, True),
}
_EXTRA: dict = {}


def algorithm_ids() -> list[str]:
    return [f"{k}-b200" for k in _GRID_ALGOS]


def register_algorithm(id: str, fn: Callable) -> None:
    """Registered ids are consulted before the built-ins (algorithms.cpp:64-67, 95-97)."""
    _EXTRA[id] = fn


def make_algorithm(id: str, options=None) -> Optional[Callable]:
    if id in _EXTRA:
        return _EXTRA[id]
    base = id[:-5] if id.endswith("-b200") else None
    if base is None or base not in _GRID_ALGOS:
        return None
    shortest, kernel, improved = _GRID_ALGOS[base]

    def run(g: BipartiteCsr, init: MatchingState, schedule=None) -> AlgorithmResult:
        if shortest:
            r = apsb(g, init, None, schedule, kernel, improved)
        else:
            r = apfb(g, init, None, schedule, kernel)
        return AlgorithmResult(r.matching, r.counters)

    return run


# ---- generators (include/bmatch_b200_gen.h) --------------------------------
def _gen(nc: int, nr: int, capacity: int, call) -> BipartiteCsr:
    cx = np.zeros(nc + 1, np.int64)
    adj = np.zeros(max(capacity, 1), np.int32)
    ne = C.c_int64()
    check(call(i64p(cx), i32p(adj), C.byref(ne)))
    return BipartiteCsr(nc, nr, cx, adj[: ne.value].copy() if ne.value < len(adj) // 2 else adj[: ne.value])


def generate_random_bipartite(nc: int, nr: int, avg_degree: float, seed: int, threads: int = 0) -> BipartiteCsr:
    """Bit-identical to the reference generator (csr_graph.cpp:92-112)."""
    cap = int(lib.bm_gen_uniform_capacity(nc, avg_degree))
    return _gen(max(nc, 0), max(nr, 0), cap,
                lambda cx, adj, ne: lib.bm_gen_uniform(nc, nr, avg_degree, seed, threads, cx, adj, ne))


def generate_planted(n: int, avg_degree: float, seed: int, threads: int = 0) -> BipartiteCsr:
    cap = int(lib.bm_gen_planted_capacity(n, avg_degree))
    return _gen(n, n, cap, lambda cx, adj, ne: lib.bm_gen_planted(n, avg_degree, seed, threads, cx, adj, ne))


def generate_rmat(scale: int, edge_factor: float, seed: int, a=0.57, b=0.19, c=0.19, permute=True,
                  threads: int = 0) -> BipartiteCsr:
    cap = int(lib.bm_gen_rmat_capacity(scale, edge_factor))
    n = 1 << scale
    return _gen(n, n, cap, lambda cx, adj, ne: lib.bm_gen_rmat(scale, edge_factor, a, b, c, seed,
                                                                1 if permute else 0, threads, cx, adj, ne))


def generate_banded(n: int, band: int, delete_frac: float, seed: int, permute=True, threads: int = 0):
    """Returns (graph, live_rows); the maximum matching has exactly live_rows pairs."""
    cap = int(lib.bm_gen_banded_capacity(n, band))
    live = C.c_int64()
    g = _gen(n, n, cap, lambda cx, adj, ne: lib.bm_gen_banded(n, band, delete_frac, seed, 1 if permute else 0,
                                                               threads, cx, adj, ne, C.byref(live)))
    return g, int(live.value)


# ---- graph files (include/bmatch_b200_io.h) -------------------------------
def _mm_build(info, load) -> BipartiteCsr:
    hdr = _lib.bm_mm_header()
    line = C.c_int64(0)
    check(info(C.byref(hdr), C.byref(line)), line.value)
    nc, nr = hdr.ncols, hdr.nrows
    return _gen(nc, nr, int(hdr.capacity),
                lambda cx, adj, ne: _status_line(load, int(hdr.capacity), cx, adj, ne))


def _status_line(load, cap, cx, adj, ne):
    line = C.c_int64(0)
    st = load(cap, cx, adj, ne, C.byref(line))
    if st:
        check(st, line.value)
    return st


def read_matrix_market(text) -> BipartiteCsr:
    """read_matrix_market (matrix_market.cpp:29-99) on an in-memory stream
    (str or bytes); raises ParseError with the reference's line number."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    return _mm_build(lambda h, ln: lib.bm_mm_parse_info(data, len(data), h, ln),
                     lambda cap, cx, adj, ne, ln: lib.bm_mm_parse(data, len(data), 0, cap, cx, adj, ne, ln))


def load_matrix_market(path: str, threads: int = 0) -> BipartiteCsr:
    """load_matrix_market (matrix_market.cpp:101-108), parsed on every host
    core; the graph name is the file stem."""
    import os
    bp = os.fsencode(path)
    g = _mm_build(lambda h, ln: lib.bm_mm_info(bp, h, ln),
                  lambda cap, cx, adj, ne, ln: lib.bm_mm_load(bp, threads, cap, cx, adj, ne, ln))
    g.name = os.path.splitext(os.path.basename(path))[0]
    return g


def write_matrix_market(g: BipartiteCsr, path: str, threads: int = 0) -> None:
    """The bytes of write_matrix_market (matrix_market.cpp:111-118)."""
    import os
    check(lib.bm_mm_write(os.fsencode(path), g.nc, g.nr, i64p(g.cxadj), i32p(g.cadj), threads))


def save_csc(g: BipartiteCsr, path: str, threads: int = 0) -> None:
    """Binary CSC container BMCSC001 (include/bmatch_b200_io.h)."""
    import os
    check(lib.bm_csc_write(os.fsencode(path), g.nc, g.nr, i64p(g.cxadj), i32p(g.cadj), threads))


def load_csc(path: str, threads: int = 0) -> BipartiteCsr:
    """Reads a BMCSC001 file; verifies its checksum and the CSC invariants."""
    import os
    bp = os.fsencode(path)
    nc, nr, ne = C.c_int32(), C.c_int32(), C.c_int64()
    check(lib.bm_csc_info(bp, C.byref(nc), C.byref(nr), C.byref(ne)))
    cx = np.zeros(nc.value + 1, np.int64)
    adj = np.zeros(max(ne.value, 1), np.int32)
    check(lib.bm_csc_read(bp, threads, ne.value, i64p(cx), i32p(adj)))
    g = BipartiteCsr(nc.value, nr.value, cx, adj[: ne.value])
    g.name = os.path.splitext(os.path.basename(path))[0]
    return g
