"""Loads libprgpu.so (the CUDA engine) and declares its C ABI (include/prgpu.h).

There is deliberately no fallback: if the library is missing or no CUDA
device is visible, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PRGPU_LIB") or os.path.join(HERE, "libprgpu.so")  # override: tuning builds

PRGPU_OK, PRGPU_EINVAL, PRGPU_ECUDA, PRGPU_ENCCL, PRGPU_ENOMEM = 0, 1, 2, 3, 4
PRGPU_EPARSE, PRGPU_EIO = 5, 6
MAX_LANES = 16

# Every symbol include/prgpu.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "prgpu_graph_build", "prgpu_graph_build_device", "prgpu_graph_from_csr",
    "prgpu_graph_generate_rmat", "prgpu_graph_generate_grid", "prgpu_graph_get_info",
    "prgpu_graph_generate_rmat_shard", "prgpu_graph_shard_info", "prgpu_device_bytes",
    "prgpu_part_need_local", "prgpu_part_set_need", "prgpu_session_kernel_times",
    "prgpu_graph_download", "prgpu_graph_free", "prgpu_pagerank", "prgpu_pagerank_observed",
    "prgpu_session_create", "prgpu_session_run", "prgpu_session_results",
    "prgpu_session_time_pull", "prgpu_session_free", "prgpu_error_norm", "prgpu_last_error",
    "prgpu_version", "prgpu_kernel_launch_count", "prgpu_part_buffer_sizes", "prgpu_part_create",
    "prgpu_part_plan", "prgpu_part_exchange", "prgpu_part_set_stream", "prgpu_part_init",
    "prgpu_part_step", "prgpu_part_finalize", "prgpu_part_active", "prgpu_part_local_ranks",
    "prgpu_part_local_ranks_device", "prgpu_part_set_peers", "prgpu_part_launch",
    "prgpu_ipc_export", "prgpu_ipc_open", "prgpu_ipc_close",
    "prgpu_graph_permutation", "prgpu_graph_rows",
    "prgpu_mtx_parse", "prgpu_mtx_load", "prgpu_pairs_free", "prgpu_graph_load_mtx",
    "prgpu_part_sent_rows", "prgpu_part_owned_ranks_device", "prgpu_pagerank_series",
]


class Partition(C.Structure):
    _fields_ = [("row_begin", C.c_uint32), ("row_end", C.c_uint32), ("src_begin", C.c_uint64),
                ("src_end", C.c_uint64), ("task_begin", C.c_uint32), ("task_end", C.c_uint32)]


class Exchange(C.Structure):
    _fields_ = [("contrib", C.c_void_p * 2), ("stride", C.c_uint32), ("nsrc", C.c_uint64),
                ("rank_partials", C.c_void_p), ("partials_per_rank", C.c_uint32)]


class GraphInfo(C.Structure):
    _fields_ = [("vertex_count", C.c_uint32), ("edge_count", C.c_uint64),
                ("dangling_count", C.c_uint32), ("max_in_degree", C.c_uint32),
                ("hub_rows", C.c_uint32), ("warp_rows", C.c_uint32),
                ("thread_rows", C.c_uint32), ("empty_rows", C.c_uint32), ("device", C.c_int)]


class Params(C.Structure):
    _fields_ = [("lanes", C.c_int), ("alphas", C.POINTER(C.c_double)),
                ("tolerances", C.POINTER(C.c_double)), ("tolerance", C.c_double),
                ("norm", C.c_int), ("stop_mask", C.c_uint32), ("max_iterations", C.c_int),
                ("ref_ranks", C.POINTER(C.c_double))]


class Result(C.Structure):
    _fields_ = [("ranks", C.POINTER(C.c_double)), ("iterations", C.POINTER(C.c_int)),
                ("converged", C.POINTER(C.c_uint8)), ("final_err", C.POINTER(C.c_double)),
                ("err_trace", C.POINTER(C.c_double)), ("loop_ms", C.c_double),
                ("run_iterations", C.c_int)]


OBSERVER = C.CFUNCTYPE(None, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_uint64, C.c_double,
                       C.c_void_p)

_lock = threading.Lock()
_lib = None


def lib():
    """The loaded library (raises if it was not built — no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; "
                               "g.build()'` (the CUDA engine has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64, i32, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
        pp = C.POINTER(vp)
        sig = {
            "prgpu_graph_build": ([u32, vp, u64, i32, pp], i32),
            "prgpu_graph_build_device": ([u32, vp, u64, i32, pp], i32),
            "prgpu_graph_from_csr": ([u32, vp, vp, vp, i32, pp], i32),
            "prgpu_graph_generate_rmat": ([u32, u32, dbl, dbl, dbl, u64, i32, pp], i32),
            "prgpu_graph_generate_grid": ([u32, dbl, dbl, u64, i32, pp], i32),
            "prgpu_graph_generate_rmat_shard": ([u32, u32, dbl, dbl, dbl, u64, i32, i32, i32, pp], i32),
            "prgpu_device_bytes": ([vp, vp, C.POINTER(u64), C.POINTER(u64)], i32),
            "prgpu_part_need_local": ([vp, vp], i32),
            "prgpu_session_kernel_times": ([vp, C.POINTER(dbl), i32, C.POINTER(i32)], i32),
            "prgpu_part_set_need": ([vp, vp], i32),
            "prgpu_graph_shard_info": ([vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(u32), C.POINTER(u32),
                                        C.POINTER(u64)], i32),
            "prgpu_graph_get_info": ([vp, C.POINTER(GraphInfo)], i32),
            "prgpu_graph_download": ([vp, vp, vp, vp, vp], i32),
            "prgpu_graph_free": ([vp], None),
            "prgpu_pagerank": ([vp, C.POINTER(Params), C.POINTER(Result)], i32),
            "prgpu_pagerank_observed": ([vp, C.POINTER(Params), C.POINTER(Result), OBSERVER, vp],
                                        i32),
            "prgpu_session_create": ([vp, C.POINTER(Params), pp], i32),
            "prgpu_session_run": ([vp, C.POINTER(dbl)], i32),
            "prgpu_session_results": ([vp, C.POINTER(Result)], i32),
            "prgpu_session_time_pull": ([vp, i32, C.POINTER(dbl)], i32),
            "prgpu_session_free": ([vp], None),
            "prgpu_error_norm": ([i32, vp, vp, u64, i32, C.POINTER(dbl)], i32),
            "prgpu_last_error": ([], C.c_char_p),
            "prgpu_version": ([], C.c_char_p),
            "prgpu_kernel_launch_count": ([], u64),
            "prgpu_part_buffer_sizes": ([vp, C.POINTER(Params), i32, C.POINTER(u64), C.POINTER(u64)], i32),
            "prgpu_part_create": ([vp, C.POINTER(Params), i32, i32, vp, vp, pp], i32),
            "prgpu_part_plan": ([vp, C.POINTER(Partition)], i32),
            "prgpu_part_exchange": ([vp, C.POINTER(Exchange)], i32),
            "prgpu_part_set_stream": ([vp, vp], i32),
            "prgpu_part_init": ([vp], i32),
            "prgpu_part_step": ([vp, C.POINTER(i32)], i32),
            "prgpu_part_finalize": ([vp], i32),
            "prgpu_part_active": ([vp, C.POINTER(i32)], i32),
            "prgpu_part_local_ranks": ([vp, i32, vp], i32),
            "prgpu_part_local_ranks_device": ([vp, vp, u64], i32),
            "prgpu_part_set_peers": ([vp, i32, vp, vp, vp, vp], i32),
            "prgpu_part_launch": ([vp], i32),
            "prgpu_ipc_export": ([vp, vp, C.POINTER(u64)], i32),
            "prgpu_ipc_open": ([vp, u64, i32, C.POINTER(vp)], i32),
            "prgpu_ipc_close": ([vp, u64], i32),
            "prgpu_graph_permutation": ([vp, vp], i32),
            "prgpu_graph_rows": ([vp, vp, C.c_uint32, vp, vp, C.c_uint64, vp], i32),
            "prgpu_mtx_parse": ([C.c_char_p, C.c_uint64, i32, vp, vp, vp, vp], i32),
            "prgpu_mtx_load": ([C.c_char_p, i32, vp, vp, vp, vp], i32),
            "prgpu_pairs_free": ([vp], None),
            "prgpu_graph_load_mtx": ([C.c_char_p, i32, i32, vp, vp], i32),
            "prgpu_part_sent_rows": ([vp, vp, vp], i32),
            "prgpu_part_owned_ranks_device": ([vp, vp, u64, vp], i32),
            "prgpu_pagerank_series": ([vp, vp, vp], i32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
        return L


def check(status: int, what: str = "") -> None:
    """Maps a PRGPU_* status to the reference's exception types."""
    if status == PRGPU_OK:
        return
    msg = lib().prgpu_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == PRGPU_EINVAL:
        raise ValueError(msg)          # std::invalid_argument
    if status == PRGPU_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)            # std::runtime_error


def default_device() -> int:
    for var in ("PRGPU_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(var)
        if v is not None and v.strip().isdigit():
            return int(v)
    return 0


def launch_count() -> int:
    return int(lib().prgpu_kernel_launch_count())
