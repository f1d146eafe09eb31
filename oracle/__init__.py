"""CPU oracle for the B200 matching engine — TEST INFRASTRUCTURE ONLY.

Two checkers, both CPU:
  * ``Oracle`` — liboracle.so, a plain-C restatement of the reference path
    (bm_oracle.c; every function cites the reference file:line it follows).
  * ``Reference`` — oracle/_ref/libbmatch_ref.so, the reference's own sources
    (/root/reference/proj/src) compiled unmodified by ``make ref`` plus a thin
    C wrapper (ref_capi.cpp). Built only where /root/reference exists; the
    prebuilt .so travels to the GPU box with the snapshot.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker or the CPU baseline —
never as the measured or shipped path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_PATH = os.path.join(_HERE, "liboracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libbmatch_ref.so")

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


def _p32(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_i32p)


def _p64(a):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


class or_graph(C.Structure):
    _fields_ = [("nc", C.c_int32), ("nr", C.c_int32), ("cxadj", _i64p), ("cadj", _i32p)]


class or_counters(C.Structure):
    _fields_ = [("outer_iterations", C.c_int64), ("columns_scanned", C.c_int64),
                ("alternations_attempted", C.c_int64), ("fix_resets", C.c_int64),
                ("serial_retries", C.c_int64), ("bfs_launches_total", C.c_int64),
                ("launches", _i64p), ("launches_cap", C.c_int64)]


class Oracle:
    """C restatement (bm_oracle.c)."""

    def __init__(self, path: str = ORACLE_PATH):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make`")
        L = self.lib = C.CDLL(path)
        G = C.POINTER(or_graph)
        sig = {
            "or_cheap_matching": (None, [G, _i32p, _i32p]),
            "or_cardinality": (C.c_int64, [C.c_int32, _i32p]),
            "or_validate": (C.c_int64, [G, _i32p, _i32p]),
            "or_is_maximum": (C.c_int32, [G, _i32p, _i32p]),
            "or_brute_force_maximum": (C.c_int64, [G]),
            "or_hopcroft_karp": (None, [G, _i32p, _i32p]),
            "or_alternating_bfs_depths": (None, [G, _i32p, _i32p, _i32p]),
            "or_init_bfs_array": (None, [C.c_int32, _i32p, C.c_int32, _i32p]),
            "or_init_root": (None, [C.c_int32, _i32p, _i32p]),
            "or_gpubfs": (C.c_int64, [G, C.c_int32, C.c_int32, C.c_int32, _i32p, _i32p, _i32p, _i32p]),
            "or_gpubfs_wr": (C.c_int64, [G, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _i32p, _i32p, _i32p,
                                         _i32p, _i32p]),
            "or_alternate": (C.c_int64, [G, C.c_int32, _i32p, _i32p, _i32p]),
            "or_alternate_wr": (C.c_int64, [G, C.c_int32, _i32p, _i32p, _i32p, _i32p]),
            "or_fix_matching": (C.c_int64, [C.c_int32, C.c_int32, _i32p, _i32p]),
            "or_driver": (C.c_int32, [G, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _i32p, _i32p,
                                      C.POINTER(or_counters)]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a

    @staticmethod
    def graph(g) -> or_graph:
        return or_graph(g.nc, g.nr, _p64(g.cxadj), _p32(g.cadj))

    def cheap_matching(self, g):
        r = np.zeros(g.nr, np.int32)
        c = np.zeros(g.nc, np.int32)
        self.lib.or_cheap_matching(C.byref(self.graph(g)), _p32(r), _p32(c))
        return r, c

    def validate(self, g, rmatch, cmatch) -> int:
        return int(self.lib.or_validate(C.byref(self.graph(g)), _p32(rmatch), _p32(cmatch)))

    def is_maximum(self, g, rmatch, cmatch) -> int:
        return int(self.lib.or_is_maximum(C.byref(self.graph(g)), _p32(rmatch), _p32(cmatch)))

    def brute_force_maximum(self, g) -> int:
        return int(self.lib.or_brute_force_maximum(C.byref(self.graph(g))))

    def hopcroft_karp(self, g, rmatch=None, cmatch=None):
        if rmatch is None:
            rmatch, cmatch = self.cheap_matching(g)
        rmatch, cmatch = rmatch.copy(), cmatch.copy()
        self.lib.or_hopcroft_karp(C.byref(self.graph(g)), _p32(rmatch), _p32(cmatch))
        return rmatch, cmatch

    def maximum(self, g) -> int:
        r, _ = self.hopcroft_karp(g)
        return int(np.count_nonzero(r >= 0))

    def depths(self, g, rmatch, cmatch):
        d = np.zeros(g.nc, np.int32)
        self.lib.or_alternating_bfs_depths(C.byref(self.graph(g)), _p32(rmatch), _p32(cmatch), _p32(d))
        return d

    def driver(self, g, rmatch, cmatch, *, tot=65536, shortest=False, kernel=1, improved=False):
        """Serial-schedule apfb/apsb. Returns (status, rmatch, cmatch, counters dict)."""
        r, c = rmatch.copy(), cmatch.copy()
        launches = np.zeros(g.nc + 2, np.int64)
        ct = or_counters()
        ct.launches = _p64(launches)
        ct.launches_cap = len(launches)
        st = self.lib.or_driver(C.byref(self.graph(g)), tot, 1 if shortest else 0, kernel, 1 if improved else 0,
                                _p32(r), _p32(c), C.byref(ct))
        n = int(ct.outer_iterations)
        d = dict(outer_iterations=n, columns_scanned=int(ct.columns_scanned),
                 alternations_attempted=int(ct.alternations_attempted), fix_resets=int(ct.fix_resets),
                 serial_retries=int(ct.serial_retries), bfs_launches_total=int(ct.bfs_launches_total),
                 bfs_launches_per_iteration=[int(x) for x in launches[:min(n, len(launches))]])
        return int(st), r, c, d


class Reference:
    """The reference library itself (oracle/_ref/libbmatch_ref.so)."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make ref` where /root/reference exists")
        # The reference's iostream-based Matrix Market reader needs the shared
        # libstdc++'s locale machinery visible globally (this toolchain links a
        # static copy into the .so; without the preload its streams crash).
        C.CDLL("libstdc++.so.6", mode=C.RTLD_GLOBAL)
        L = self.lib = C.CDLL(path)
        vp = C.c_void_p
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_hw_threads": (C.c_int32, []),
            "ref_graph_from_csc": (vp, [C.c_int32, C.c_int32, _i64p, _i32p]),
            "ref_generate_random_bipartite": (vp, [C.c_int32, C.c_int32, C.c_double, C.c_uint64]),
            "ref_permute_random": (vp, [vp, C.c_uint64]),
            "ref_graph_info": (None, [vp, _i32p, _i32p, _i64p]),
            "ref_graph_copy": (None, [vp, _i64p, _i32p]),
            "ref_graph_free": (None, [vp]),
            "ref_check_csr": (C.c_int32, [vp]),
            "ref_cheap_matching": (None, [vp, _i32p, _i32p]),
            "ref_brute_force_maximum": (C.c_int64, [vp]),
            "ref_validate": (C.c_int64, [vp, _i32p, _i32p]),
            "ref_is_maximum": (C.c_int32, [vp, _i32p, _i32p]),
            "ref_run": (C.c_int32, [vp, C.c_char_p, C.c_char_p, C.c_int32, _i32p, _i32p, _i64p, _i64p, C.c_int64,
                                    C.POINTER(C.c_double)]),
            "ref_gpubfs": (C.c_int64, [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _i32p, _i32p, _i32p, _i32p,
                                       _i32p, _i32p]),
            "ref_alternate": (C.c_int64, [vp, C.c_int32, C.c_int32, _i32p, _i32p, _i32p, _i32p]),
            "ref_fix_matching": (C.c_int64, [C.c_int32, C.c_int32, _i32p, _i32p]),
            "ref_read_matrix_market": (vp, [C.c_char_p, C.c_int64, _i32p, _i64p]),
            "ref_write_matrix_market": (C.c_int64, [vp, C.c_char_p, C.c_int64]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a

    def error(self) -> str:
        return (self.lib.ref_last_error() or b"").decode()

    def hw_threads(self) -> int:
        return int(self.lib.ref_hw_threads())

    # graphs are handles owned by the reference library
    def from_csc(self, g):
        return RefGraph(self, self.lib.ref_graph_from_csc(g.nc, g.nr, _p64(g.cxadj), _p32(g.cadj)))

    def generate_random_bipartite(self, nc, nr, deg, seed):
        return RefGraph(self, self.lib.ref_generate_random_bipartite(nc, nr, deg, seed))

    def read_matrix_market(self, text: bytes):
        """-> ("ok", nc, nr, cxadj, cadj) | ("parse", line, message) | ("error", message)."""
        kind, line = C.c_int32(), C.c_int64()
        h = self.lib.ref_read_matrix_market(text, len(text), C.byref(kind), C.byref(line))
        if not h:
            return ("parse", line.value, self.error()) if kind.value == 1 else ("error", self.error())
        return ("ok",) + RefGraph(self, h).arrays()

    def write_matrix_market(self, g) -> bytes:
        rg = self.from_csc(g)
        n = self.lib.ref_write_matrix_market(rg.h, None, 0)
        buf = C.create_string_buffer(max(n, 1))
        self.lib.ref_write_matrix_market(rg.h, buf, n)
        return buf.raw[:n]

    def fix_matching(self, rmatch, cmatch):
        r, c = rmatch.copy(), cmatch.copy()
        n = self.lib.ref_fix_matching(len(c), len(r), _p32(r), _p32(c))
        return int(n), r, c


class RefGraph:
    def __init__(self, ref: Reference, handle):
        self.ref, self.h = ref, handle

    def __del__(self):
        try:
            self.ref.lib.ref_graph_free(self.h)
        except Exception:
            pass

    def info(self):
        nc, nr, ne = C.c_int32(), C.c_int32(), C.c_int64()
        self.ref.lib.ref_graph_info(self.h, C.byref(nc), C.byref(nr), C.byref(ne))
        return nc.value, nr.value, ne.value

    def arrays(self):
        nc, nr, ne = self.info()
        cx = np.zeros(nc + 1, np.int64)
        adj = np.zeros(max(ne, 1), np.int32)
        self.ref.lib.ref_graph_copy(self.h, _p64(cx), _p32(adj))
        return nc, nr, cx, adj[:ne]

    def permute(self, seed):
        return RefGraph(self.ref, self.ref.lib.ref_permute_random(self.h, seed))

    def cheap_matching(self):
        nc, nr, _ = self.info()
        r = np.zeros(nr, np.int32)
        c = np.zeros(nc, np.int32)
        self.ref.lib.ref_cheap_matching(self.h, _p32(r), _p32(c))
        return r, c

    def brute_force_maximum(self):
        return int(self.ref.lib.ref_brute_force_maximum(self.h))

    def validate(self, r, c):
        return int(self.ref.lib.ref_validate(self.h, _p32(r), _p32(c)))

    def is_maximum(self, r, c):
        return int(self.ref.lib.ref_is_maximum(self.h, _p32(r), _p32(c)))

    def run(self, algo: str, rmatch, cmatch, schedule="serial", ct_threads=0):
        """make_algorithm(algo)(g, init, parse_schedule(schedule)). Returns (rmatch, cmatch, counters, seconds)."""
        r, c = rmatch.copy(), cmatch.copy()
        nc = len(c)
        counters = np.zeros(6, np.int64)
        launches = np.zeros(nc + 2, np.int64)
        secs = C.c_double()
        st = self.ref.lib.ref_run(self.h, algo.encode(), schedule.encode(), ct_threads, _p32(r), _p32(c),
                                  _p64(counters), _p64(launches), len(launches), C.byref(secs))
        if st != 0:
            raise RuntimeError(f"reference run failed ({st}): {self.ref.error()}")
        d = dict(outer_iterations=int(counters[0]), columns_scanned=int(counters[1]),
                 alternations_attempted=int(counters[2]), fix_resets=int(counters[3]),
                 serial_retries=int(counters[4]), bfs_launches_total=int(counters[5]),
                 bfs_launches_per_iteration=[int(x) for x in launches[:int(counters[0])]])
        return r, c, d, secs.value


def have_reference() -> bool:
    return os.path.exists(REF_PATH)


GEN_PATH = os.path.join(_HERE, "libgen_oracle.so")


class OGraph:
    """A CSC in numpy arrays, shaped like paper_1303_1379_b200.BipartiteCsr
    (nc, nr, cxadj int64, cadj int32) but built without the product library."""

    def __init__(self, nc, nr, cxadj, cadj, name=""):
        self.nc, self.nr, self.cxadj, self.cadj, self.name = nc, nr, cxadj, cadj, name

    def num_edges(self) -> int:
        return int(self.cxadj[-1])


class Generators:
    """gen_oracle.cpp: the bench configs' synthetic graphs restated for the
    reference arm / CPU baseline (the product's generators live in libbmatch_b200.so)."""

    def __init__(self, path: str = GEN_PATH, threads: int = 0):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make`")
        L = self.lib = C.CDLL(path)
        self.threads = threads
        i32, i64, dbl, u64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64
        sig = {
            "go_uniform": [i32, i32, dbl, u64, i32, _i64p, _i32p],
            "go_planted": [i32, dbl, u64, i32, _i64p, _i32p],
            "go_rmat": [i32, dbl, dbl, dbl, dbl, u64, i32, i32, _i64p, _i32p],
            "go_banded": [i32, i32, dbl, u64, i32, i32, _i64p, _i32p, _i64p],
        }
        for k, a in sig.items():
            getattr(L, k).restype = C.c_int64
            getattr(L, k).argtypes = a
        L.go_first_fit.restype = None
        L.go_first_fit.argtypes = [i32, i32, _i64p, _i32p, _i32p, _i32p]

    @staticmethod
    def _alloc(nc, cap):
        return np.empty(nc + 1, np.int64), np.empty(max(int(cap), 1), np.int32)

    def _done(self, nc, nr, cx, adj, ne, name):
        return OGraph(nc, nr, cx, adj[:ne], name)

    def uniform(self, nc, nr, deg, seed):
        cx, adj = self._alloc(nc, round(nc * deg))
        ne = self.lib.go_uniform(nc, nr, deg, seed, self.threads, _p64(cx), _p32(adj))
        return self._done(nc, nr, cx, adj, ne, f"uniform/{nc}/{deg}/{seed}")

    def planted(self, n, deg, seed):
        cx, adj = self._alloc(n, n + max(0, round((deg - 1.0) * n)))
        ne = self.lib.go_planted(n, deg, seed, self.threads, _p64(cx), _p32(adj))
        return self._done(n, n, cx, adj, ne, f"planted/{n}/{deg}/{seed}")

    def rmat(self, scale, ef, seed, a=0.57, b=0.19, c=0.19, permute=True):
        n = 1 << scale
        cx, adj = self._alloc(n, round(ef * n))
        ne = self.lib.go_rmat(scale, ef, a, b, c, seed, 1 if permute else 0, self.threads, _p64(cx), _p32(adj))
        return self._done(n, n, cx, adj, ne, f"rmat/{scale}/{ef}/{seed}")

    def banded(self, n, band, frac, seed, permute=True):
        cx, adj = self._alloc(n, n * band)
        live = C.c_int64()
        ne = self.lib.go_banded(n, band, frac, seed, 1 if permute else 0, self.threads, _p64(cx), _p32(adj),
                                C.byref(live))
        return self._done(n, n, cx, adj, ne, f"banded/{n}/{band}/{frac}/{seed}"), int(live.value)

    def first_fit(self, g):
        r = np.empty(g.nr, np.int32)
        c = np.empty(g.nc, np.int32)
        self.lib.go_first_fit(g.nc, g.nr, _p64(g.cxadj), _p32(g.cadj), _p32(r), _p32(c))
        return r, c
