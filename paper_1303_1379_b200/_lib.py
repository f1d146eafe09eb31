"""ctypes binding of the C ABI in include/bmatch_b200.h and include/bmatch_b200_gen.h.

This is the reference-side binding a Python caller would add: plain pointers
and sizes, no torch types. The library is built in-tree
(``make`` -> paper_1303_1379_b200/libbmatch_b200.so); importing this module
without it raises immediately — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BM_LIB") or os.path.join(_HERE, "libbmatch_b200.so")  # BM_LIB: alternative build (tuning)
HEADERS = [
    os.path.join(os.path.dirname(_HERE), "include", "bmatch_b200.h"),
    os.path.join(os.path.dirname(_HERE), "include", "bmatch_b200_gen.h"),
    os.path.join(os.path.dirname(_HERE), "include", "bmatch_b200_io.h"),
]

BM_OK = 0
BM_ERR_INVALID_ARG = 1
BM_ERR_LOGIC = 2
BM_ERR_BOUND_EXCEEDED = 3
BM_ERR_CUDA = 4
BM_ERR_OOM = 5
BM_ERR_NCCL = 6
BM_ERR_PARSE = 7
BM_ERR_IO = 8

BM_DRIVER_APFB, BM_DRIVER_APSB = 0, 1
BM_BFS_GPUBFS, BM_BFS_WR = 0, 1
BM_INIT_GIVEN, BM_INIT_GPU_GREEDY, BM_INIT_GPU_KS = 0, 1, 2
BM_CLAIM_REFERENCE, BM_CLAIM_AT_DISCOVERY = 0, 1
BM_EP_AUTO, BM_EP_EVERY, BM_EP_ONE_PER_TREE = 0, 1, 2
BM_BU_OFF, BM_BU_ON, BM_BU_AUTO = 0, 1, 2


class bm_match_opts(C.Structure):
    _fields_ = [
        ("driver", C.c_int32),
        ("bfs_kernel", C.c_int32),
        ("improved", C.c_int32),
        ("init", C.c_int32),
        ("max_phases", C.c_int32),
        ("claim_policy", C.c_int32),
        ("endpoint_policy", C.c_int32),
        ("bottom_up", C.c_int32),
    ]


class bm_counters(C.Structure):
    _fields_ = [
        ("outer_iterations", C.c_int64),
        ("bfs_launches_total", C.c_int64),
        ("columns_scanned", C.c_int64),
        ("alternations_attempted", C.c_int64),
        ("fix_resets", C.c_int64),
        ("serial_retries", C.c_int64),
        ("edges_traversed", C.c_int64),
        ("columns_visited", C.c_int64),
        ("walk_steps", C.c_int64),
        ("frontier_entries", C.c_int64),
        ("cardinality", C.c_int64),
        ("initial_cardinality", C.c_int64),
        ("n_phase_records", C.c_int64),
        ("reserved", C.c_int64 * 3),
    ]


class bm_phase_event(C.Structure):
    _fields_ = [
        ("iteration", C.c_int64),
        ("augmenting_path_found", C.c_int32),
        ("serial_retry", C.c_int32),
        ("cardinality_before", C.c_int64),
        ("cardinality_after", C.c_int64),
        ("bfs_launches", C.c_int64),
        ("rmatch", C.POINTER(C.c_int32)),
        ("nr", C.c_int32),
        ("cmatch", C.POINTER(C.c_int32)),
        ("nc", C.c_int32),
    ]


class bm_mm_header(C.Structure):
    _fields_ = [
        ("nrows", C.c_int32),
        ("ncols", C.c_int32),
        ("entries", C.c_int64),
        ("symmetric", C.c_int32),
        ("field", C.c_int32),
        ("capacity", C.c_int64),
    ]


PHASE_CB = C.CFUNCTYPE(C.c_int, C.POINTER(bm_phase_event), C.c_void_p)

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_vp = C.c_void_p

_PROTOS = {
    "bm_abi_version": (C.c_int32, []),
    "bm_last_error": (C.c_char_p, []),
    "bm_status_string": (C.c_char_p, [C.c_int32]),
    "bm_device_count": (C.c_int32, []),
    "bm_create": (C.c_int, [C.c_int32, C.POINTER(_vp)]),
    "bm_destroy": (C.c_int, [_vp]),
    "bm_set_stream": (C.c_int, [_vp, _vp]),
    "bm_upload_csc": (C.c_int, [_vp, C.c_int32, C.c_int32, _i64p, _i32p]),
    "bm_graph_info": (C.c_int, [_vp, _i32p, _i32p, _i64p]),
    "bm_bottom_up_auto": (C.c_int, [_vp, _i32p]),
    "bm_prepare_row_index": (C.c_int, [_vp]),
    "bm_download_row_index": (C.c_int, [_vp, C.POINTER(C.c_uint32), _i32p]),
    "bm_last_phase_launches": (C.c_int, [_vp, _i64p, C.c_int64, _i64p]),
    "bm_match": (C.c_int, [_vp, C.POINTER(bm_match_opts), _i32p, _i32p, _i64p, C.POINTER(bm_counters),
                           _i64p, C.c_int64, PHASE_CB, _vp]),
    "bm_load_matching": (C.c_int, [_vp, _i32p, _i32p]),
    "bm_run": (C.c_int, [_vp, C.POINTER(bm_match_opts), _i64p, C.POINTER(bm_counters), _i64p, C.c_int64,
                         PHASE_CB, _vp, _i32p]),
    "bm_resume": (C.c_int, [_vp, C.POINTER(bm_match_opts), _i64p, C.POINTER(bm_counters), _i64p, C.c_int64,
                            PHASE_CB, _vp, _i32p]),
    "bm_download_matching": (C.c_int, [_vp, _i32p, _i32p]),
    "bm_last_kernel_time": (C.c_int, [_vp, C.POINTER(C.c_double), _i32p]),
    "bm_debug_set": (C.c_int, [_vp, C.c_int32, C.c_int64]),
    "bm_timeline": (C.c_int, [_vp, C.POINTER(C.c_uint64), C.c_int64, _i64p]),
    "bm_debug_stats": (C.c_int, [_vp, C.POINTER(C.c_uint64), C.c_int64, _i64p]),
    "bm_bfs_phase": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, _i32p, _i32p, _i32p, _i32p, _i32p,
                               _i64p, _i32p]),
    "bm_verify": (C.c_int, [_vp, _i32p, _i32p, _i64p, _i32p, _i64p]),
    "bm_permute_random": (C.c_int, [_vp, _i32p, _i32p]),
    "bm_download_csc": (C.c_int, [_vp, _i64p, _i32p]),
    "bm_permutation_pair": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, _i32p, _i32p]),
    "bm_host_cheap_matching": (C.c_int, [C.c_int32, C.c_int32, _i64p, _i32p, _i32p, _i32p]),
    "bm_gen_uniform_capacity": (C.c_int64, [C.c_int32, C.c_double]),
    "bm_gen_uniform": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.c_int32, _i64p, _i32p, _i64p]),
    "bm_gen_planted_capacity": (C.c_int64, [C.c_int32, C.c_double]),
    "bm_gen_planted": (C.c_int, [C.c_int32, C.c_double, C.c_uint64, C.c_int32, _i64p, _i32p, _i64p]),
    "bm_gen_rmat_capacity": (C.c_int64, [C.c_int32, C.c_double]),
    "bm_gen_rmat": (C.c_int, [C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64,
                              C.c_int32, C.c_int32, _i64p, _i32p, _i64p]),
    "bm_gen_banded_capacity": (C.c_int64, [C.c_int32, C.c_int32]),
    "bm_gen_banded": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.c_int32, C.c_int32, _i64p,
                                _i32p, _i64p, _i64p]),
    "bm_check_csc": (C.c_int, [C.c_int32, C.c_int32, _i64p, _i32p]),
    "bm_csc_digest": (C.c_uint64, [C.c_int32, C.c_int32, _i64p, _i32p]),
    "bm_mm_info": (C.c_int, [C.c_char_p, C.POINTER(bm_mm_header), _i64p]),
    "bm_mm_load": (C.c_int, [C.c_char_p, C.c_int32, C.c_int64, _i64p, _i32p, _i64p, _i64p]),
    "bm_mm_parse_info": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(bm_mm_header), _i64p]),
    "bm_mm_parse": (C.c_int, [C.c_char_p, C.c_int64, C.c_int32, C.c_int64, _i64p, _i32p, _i64p, _i64p]),
    "bm_mm_write": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, _i64p, _i32p, C.c_int32]),
    "bm_csc_write": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, _i64p, _i32p, C.c_int32]),
    "bm_csc_info": (C.c_int, [C.c_char_p, _i32p, _i32p, _i64p]),
    "bm_csc_read": (C.c_int, [C.c_char_p, C.c_int32, C.c_int64, _i64p, _i32p]),
}


def declared_symbols() -> list[str]:
    """Function names declared in include/*.h (the ABI surface)."""
    names = []
    for path in HEADERS:
        text = open(path).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s+\**\s*(bm_[a-z0-9_]+)\s*\(",
                             text, flags=re.M):
            names.append(m.group(1))
    return sorted(set(names))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a engine with `make` (or __graft_entry__.build()). "
            "There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _PROTOS.items():
        if os.environ.get("BM_LIB") and not hasattr(lib, name):
            continue  # an older tuning build (BM_LIB) may lack newer entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class LogicError(Exception):
    """Mirror of std::logic_error (gpu_match.cpp:77-80, 272-274)."""


class ParseError(ValueError):
    """Mirror of bmatch::ParseError (parse_error.hpp:9-14): a malformed input
    file, tagged with the 1-based line number."""

    def __init__(self, line: int, message: str):
        super().__init__(message)
        self.line = line


class CudaError(RuntimeError):
    """The device path failed (no GPU, launch error, out of memory)."""


def check(status: int, line: int = 0) -> None:
    if status == BM_OK:
        return
    msg = (lib.bm_last_error() or b"").decode(errors="replace")
    name = (lib.bm_status_string(status) or b"").decode()
    text = f"{name}: {msg}"
    if status == BM_ERR_PARSE:
        raise ParseError(line, msg)
    if status == BM_ERR_IO:
        raise OSError(msg)
    if status == BM_ERR_INVALID_ARG:
        raise ValueError(text)
    if status == BM_ERR_LOGIC:
        raise LogicError(text)
    if status == BM_ERR_BOUND_EXCEEDED:
        raise RuntimeError(text)
    if status == BM_ERR_OOM:
        raise MemoryError(text)
    raise CudaError(text)


def i32p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_i32p)


def i64p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)
