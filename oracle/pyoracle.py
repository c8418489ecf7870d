"""ctypes bindings for the TEST-ONLY checkers in oracle/.

    Oracle   — oracle/liboracle.so, the C restatement (oracle.c)
    Ref      — oracle/_ref/libprref.so, the reference's own headers behind a C shim

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
legs may import this module.  The product (paper_2108_02997_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libprref.so")

NORMS = {"l1": 0, "l2": 1, "linf": 2}

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> None:
    """Compile the checkers (make -C oracle)."""
    if force or not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def _norm_id(norm) -> int:
    return NORMS[norm] if isinstance(norm, str) else int(norm)


class _Edges(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint64), ("cap", C.c_uint64),
                ("pairs", C.POINTER(C.c_uint32))]


class _Csr(C.Structure):
    _fields_ = [("n", C.c_uint32), ("e", C.c_uint64),
                ("in_offsets", C.POINTER(C.c_uint64)),
                ("in_neighbors", C.POINTER(C.c_uint32)),
                ("out_degree", C.POINTER(C.c_uint32)),
                ("dangling", C.POINTER(C.c_uint32)),
                ("ndangling", C.c_uint32)]


class _MT(C.Structure):
    _fields_ = [("mt", C.c_uint32 * 624), ("idx", C.c_int)]


class CsrArrays:
    """Host copy of a reverse CSR in the reference layout (graph.hpp:47-60)."""

    def __init__(self, n, in_offsets, in_neighbors, out_degree, dangling):
        self.vertex_count = int(n)
        self.in_offsets = in_offsets
        self.in_neighbors = in_neighbors
        self.out_degree = out_degree
        self.dangling = dangling

    def edge_count(self) -> int:
        return int(self.in_neighbors.size)


class Oracle:
    """The C restatement (oracle/oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        build()
        L = C.CDLL(path)
        self.L = L
        L.orc_mt_seed.argtypes = [C.POINTER(_MT), C.c_uint32]
        L.orc_mt_next.argtypes = [C.POINTER(_MT)]
        L.orc_mt_next.restype = C.c_uint32
        for name, args in [
            ("orc_random_digraph", [C.POINTER(_MT), C.c_uint32, C.c_double, C.c_int]),
            ("orc_regular_ring", [C.c_uint32, C.c_uint32]),
            ("orc_scale_free_web", [C.POINTER(_MT), C.c_uint32, C.c_uint32, C.c_double]),
            ("orc_rmat", [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64]),
            ("orc_grid", [C.c_uint32, C.c_double, C.c_double, C.c_uint64]),
        ]:
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.POINTER(_Edges)
        L.orc_edges_free.argtypes = [C.POINTER(_Edges)]
        L.orc_build_csr.argtypes = [C.c_uint32, _u32p, C.c_uint64]
        L.orc_build_csr.restype = C.POINTER(_Csr)
        L.orc_csr_free.argtypes = [C.POINTER(_Csr)]
        L.orc_error_norm.argtypes = [C.c_int, _f64p, _f64p, C.c_uint64]
        L.orc_error_norm.restype = C.c_double
        L.orc_pagerank.argtypes = [C.POINTER(_Csr), C.c_double, C.c_double, C.c_int, C.c_int,
                                   _f64p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p]
        L.orc_pagerank_mt.argtypes = [C.POINTER(_Csr), C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                      C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p,
                                      C.POINTER(C.c_double)]
        L.orc_dense_pagerank.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_double, C.c_double,
                                         C.c_int, C.c_int, _f64p, C.POINTER(C.c_int),
                                         C.POINTER(C.c_int)]
        L.orc_pagerank_step_rows.argtypes = [C.c_uint32, _f64p, _u32p, C.c_double, C.c_uint32,
                                             _u64p, _u32p, _f64p]
        L.orc_pagerank_step_rows.restype = C.c_double
        L.orc_estimate_iterations.argtypes = [C.c_double, C.c_double]
        L.orc_estimate_iterations.restype = C.c_int
        L.orc_hash64.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_hash64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_mix64.restype = C.c_uint64
        L.orc_rmat_perm.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64]
        L.orc_rmat_perm.restype = C.c_uint32

    # -- rng / generators ---------------------------------------------------
    def mt19937(self, seed: int):
        s = _MT()
        self.L.orc_mt_seed(C.byref(s), seed)
        return s

    def mt_next(self, s) -> int:
        return self.L.orc_mt_next(C.byref(s))

    def _take_edges(self, p):
        e = p.contents
        pairs = np.ctypeslib.as_array(e.pairs, shape=(2 * e.m,)).copy() if e.m else \
            np.zeros(0, np.uint32)
        n = e.n
        self.L.orc_edges_free(p)
        return n, pairs

    def random_digraph(self, rng, n, p, force_dangling):
        return self._take_edges(self.L.orc_random_digraph(C.byref(rng), n, p, int(force_dangling)))

    def regular_ring(self, n, k):
        return self._take_edges(self.L.orc_regular_ring(n, k))

    def scale_free_web(self, rng, n, out_links=4, dangling_fraction=0.05):
        return self._take_edges(self.L.orc_scale_free_web(C.byref(rng), n, out_links,
                                                          dangling_fraction))

    def rmat(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1):
        return self._take_edges(self.L.orc_rmat(scale, edge_factor, a, b, c, seed))

    def grid(self, side, p=0.6, longrange_frac=0.01, seed=1):
        return self._take_edges(self.L.orc_grid(side, p, longrange_frac, seed))

    # -- csr / engine ---------------------------------------------------------
    def build_csr_handle(self, n, pairs):
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
        return self.L.orc_build_csr(n, pairs, pairs.size // 2)

    def csr_arrays(self, h) -> CsrArrays:
        g = h.contents
        n, e = g.n, g.e
        as_arr = np.ctypeslib.as_array
        return CsrArrays(
            n,
            as_arr(g.in_offsets, shape=(n + 1,)).copy(),
            as_arr(g.in_neighbors, shape=(e,)).copy() if e else np.zeros(0, np.uint32),
            as_arr(g.out_degree, shape=(n,)).copy() if n else np.zeros(0, np.uint32),
            as_arr(g.dangling, shape=(g.ndangling,)).copy() if g.ndangling else
            np.zeros(0, np.uint32))

    def build_csr(self, n, pairs) -> CsrArrays:
        h = self.build_csr_handle(n, pairs)
        try:
            return self.csr_arrays(h)
        finally:
            self.L.orc_csr_free(h)

    def free_csr(self, h):
        self.L.orc_csr_free(h)

    def pagerank(self, h, alpha=0.85, tol=1e-6, norm="l1", max_iter=500, trace=False):
        n = h.contents.n
        ranks = np.zeros(max(n, 1), np.float64)
        it, conv = C.c_int(), C.c_int()
        tr = np.zeros(max_iter, np.float64) if trace else None
        st = self.L.orc_pagerank(h, alpha, tol, _norm_id(norm), max_iter, ranks,
                                 C.byref(it), C.byref(conv),
                                 tr.ctypes.data if trace else None)
        if st != 0:
            raise ValueError("oracle pagerank: invalid argument")
        out = dict(ranks=ranks[:n], iterations=it.value, converged=bool(conv.value))
        if trace:
            out["err_trace"] = tr[: it.value]
        return out

    def csr_view(self, n, in_offsets, in_neighbors, out_degree):
        """An orc_csr over caller-owned reference-layout arrays (no copy; the
        dangling list = out_degree == 0 ascending, graph.hpp:230-231).  The
        returned object keeps the arrays alive; pass it where a handle goes."""
        off = np.ascontiguousarray(in_offsets, np.uint64)
        nbr = np.ascontiguousarray(in_neighbors, np.uint32)
        deg = np.ascontiguousarray(out_degree, np.uint32)
        dang = np.flatnonzero(deg == 0).astype(np.uint32)
        keep = (off, nbr if nbr.size else np.zeros(1, np.uint32), deg, dang if dang.size else
                np.zeros(1, np.uint32))
        c = _Csr(n, int(off[-1]), keep[0].ctypes.data_as(C.POINTER(C.c_uint64)),
                 keep[1].ctypes.data_as(C.POINTER(C.c_uint32)), keep[2].ctypes.data_as(C.POINTER(C.c_uint32)),
                 keep[3].ctypes.data_as(C.POINTER(C.c_uint32)), int(dang.size))

        class _View:
            pass
        v = _View()
        v.keep, v.csr = keep, c
        v.ptr = C.pointer(c)
        return v

    def pagerank_mt(self, view, alpha=0.85, tol=1e-6, norm="l1", max_iter=500, threads=None,
                    trace=False, want_ranks=True):
        """orc_pagerank_mt: the vertex loop on `threads` host threads, results
        bit-identical to the reference; elapsed_ms = loop time."""
        h = view.ptr if hasattr(view, "ptr") else view
        n = h.contents.n
        threads = threads or (os.cpu_count() or 1)
        ranks = np.zeros(max(n, 1), np.float64) if want_ranks else None
        it, conv, ms = C.c_int(), C.c_int(), C.c_double()
        tr = np.zeros(max_iter, np.float64) if trace else None
        st = self.L.orc_pagerank_mt(h, alpha, tol, _norm_id(norm), max_iter, threads,
                                    ranks.ctypes.data if want_ranks else None, C.byref(it), C.byref(conv),
                                    tr.ctypes.data if trace else None, C.byref(ms))
        if st != 0:
            raise ValueError("oracle pagerank_mt: invalid argument or out of memory")
        out = dict(iterations=it.value, converged=bool(conv.value), elapsed_ms=ms.value, threads=threads)
        if want_ranks:
            out["ranks"] = ranks[:n]
        if trace:
            out["err_trace"] = tr[: it.value]
        return out

    def step_rows(self, prev, out_degree, alpha, off, nbr):
        """One reference iteration (pagerank.hpp:85-93) for the rows whose
        in-neighbours are off/nbr, from the full previous vector.  Returns
        (next values [rows], teleport)."""
        prev = np.ascontiguousarray(prev, np.float64)
        deg = np.ascontiguousarray(out_degree, np.uint32)
        off = np.ascontiguousarray(off, np.uint64)
        nbr = np.ascontiguousarray(nbr if len(nbr) else np.zeros(1, np.uint32), np.uint32)
        out = np.zeros(max(len(off) - 1, 1), np.float64)
        c0 = self.L.orc_pagerank_step_rows(prev.size, prev, deg, alpha, len(off) - 1, off, nbr, out)
        return out[: len(off) - 1], c0

    def dense_pagerank(self, n, pairs, alpha, tol, norm, max_iter=500):
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
        ranks = np.zeros(n, np.float64)
        it, conv = C.c_int(), C.c_int()
        self.L.orc_dense_pagerank(n, pairs, pairs.size // 2, alpha, tol, _norm_id(norm),
                                  max_iter, ranks, C.byref(it), C.byref(conv))
        return dict(ranks=ranks, iterations=it.value, converged=bool(conv.value))

    def error_norm(self, norm, r, s) -> float:
        r = np.ascontiguousarray(r, np.float64)
        s = np.ascontiguousarray(s, np.float64)
        if r.size != s.size or r.size == 0:
            raise ValueError("error_norm: bad lengths")
        return self.L.orc_error_norm(_norm_id(norm), r, s, r.size)

    def estimate_iterations(self, alpha, tol) -> int:
        v = self.L.orc_estimate_iterations(alpha, tol)
        if v < 0:
            raise ValueError("estimate_iterations: argument outside (0, 1)")
        return v

    def hash64(self, arr: np.ndarray) -> int:
        arr = np.ascontiguousarray(arr)
        return int(self.L.orc_hash64(arr.ctypes.data, arr.nbytes))

    def mix64(self, z: int) -> int:
        return int(self.L.orc_mix64(z))


class Ref:
    """The reference's own code (oracle/_ref/libprref.so, built from /root/reference)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(force=True)
        L = C.CDLL(path)
        self.L = L
        L.ref_build_csr.argtypes = [C.c_uint32, _u32p, C.c_uint64]
        L.ref_build_csr.restype = C.c_void_p
        L.ref_csr_free.argtypes = [C.c_void_p]
        L.ref_csr_from_arrays.argtypes = [C.c_uint32, _u64p, _u32p, _u32p]
        L.ref_csr_from_arrays.restype = C.c_void_p
        L.ref_csr_rmat.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_uint64]
        L.ref_csr_rmat.restype = C.c_void_p
        L.ref_csr_vertex_count.argtypes = [C.c_void_p]
        L.ref_csr_vertex_count.restype = C.c_uint32
        L.ref_csr_edge_count.argtypes = [C.c_void_p]
        L.ref_csr_edge_count.restype = C.c_uint64
        L.ref_csr_dangling_count.argtypes = [C.c_void_p]
        L.ref_csr_dangling_count.restype = C.c_uint32
        L.ref_csr_copy.argtypes = [C.c_void_p, _u64p, _u32p, _u32p, _u32p]
        L.ref_pagerank.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, C.c_int,
                                   C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.c_void_p, C.POINTER(C.c_double)]
        L.ref_error_norm.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                     C.POINTER(C.c_int)]
        L.ref_error_norm.restype = C.c_double
        L.ref_estimate_iterations.argtypes = [C.c_double, C.c_double]
        L.ref_estimate_iterations.restype = C.c_int
        L.ref_rng_new.argtypes = [C.c_uint32]
        L.ref_rng_new.restype = C.c_void_p
        L.ref_rng_free.argtypes = [C.c_void_p]
        L.ref_rng_next.argtypes = [C.c_void_p]
        L.ref_rng_next.restype = C.c_uint32
        L.ref_gen_random_digraph.argtypes = [C.c_void_p, C.c_uint32, C.c_double, C.c_int]
        L.ref_gen_random_digraph.restype = C.c_void_p
        L.ref_gen_regular_ring.argtypes = [C.c_uint32, C.c_uint32]
        L.ref_gen_regular_ring.restype = C.c_void_p
        L.ref_gen_scale_free_web.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_double]
        L.ref_gen_scale_free_web.restype = C.c_void_p
        L.ref_edges_n.argtypes = [C.c_void_p]
        L.ref_edges_n.restype = C.c_uint32
        L.ref_edges_m.argtypes = [C.c_void_p]
        L.ref_edges_m.restype = C.c_uint64
        L.ref_edges_copy.argtypes = [C.c_void_p, _u32p]
        L.ref_edges_free.argtypes = [C.c_void_p]
        L.ref_dense_pagerank.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_double, C.c_double,
                                         C.c_int, C.c_int, _f64p, C.POINTER(C.c_int),
                                         C.POINTER(C.c_int)]

    # -- generators -------------------------------------------------------------
    def rng(self, seed):
        return self.L.ref_rng_new(seed)

    def rng_free(self, r):
        self.L.ref_rng_free(r)

    def rng_next(self, r) -> int:
        return self.L.ref_rng_next(r)

    def _take(self, h):
        n, m = self.L.ref_edges_n(h), self.L.ref_edges_m(h)
        pairs = np.zeros(2 * m, np.uint32)
        if m:
            self.L.ref_edges_copy(h, pairs)
        self.L.ref_edges_free(h)
        return n, pairs

    def random_digraph(self, rng, n, p, force_dangling):
        return self._take(self.L.ref_gen_random_digraph(rng, n, p, int(force_dangling)))

    def regular_ring(self, n, k):
        return self._take(self.L.ref_gen_regular_ring(n, k))

    def scale_free_web(self, rng, n, out_links=4, dangling_fraction=0.05):
        return self._take(self.L.ref_gen_scale_free_web(rng, n, out_links, dangling_fraction))

    # -- csr / engine -------------------------------------------------------------
    def build_csr_handle(self, n, pairs):
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
        if pairs.size == 0:
            pairs = np.zeros(2, np.uint32)
            return self.L.ref_build_csr(n, pairs, 0)
        return self.L.ref_build_csr(n, pairs, pairs.size // 2)

    def parse_mtx(self, text: bytes):
        """parse_matrix_market (graph.hpp:111-199): (n, pairs[m,2]) or raises
        ValueError((line, what))."""
        L = self.L
        L.ref_parse_mtx.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64), C.c_char_p, C.c_int]
        L.ref_parse_mtx.restype = C.c_void_p
        line = C.c_uint64()
        msg = C.create_string_buffer(512)
        h = L.ref_parse_mtx(text, len(text), C.byref(line), msg, 512)
        if not h:
            raise ValueError((int(line.value), msg.value.decode()))
        n, pairs = self._take(h)
        return n, np.asarray(pairs, np.uint32).reshape(-1, 2)

    def load_mtx(self, path: str):
        """load_matrix_market (graph.hpp:238-247): (n, pairs) or raises
        RuntimeError(what)."""
        L = self.L
        L.ref_load_mtx.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.ref_load_mtx.restype = C.c_void_p
        msg = C.create_string_buffer(4096)
        h = L.ref_load_mtx(path.encode(), msg, 4096)
        if not h:
            raise RuntimeError(msg.value.decode())
        n, pairs = self._take(h)
        return n, np.asarray(pairs, np.uint32).reshape(-1, 2)

    def free_csr(self, h):
        self.L.ref_csr_free(h)

    def csr_from_arrays(self, n, in_offsets, in_neighbors, out_degree):
        nbr = np.ascontiguousarray(in_neighbors, np.uint32)
        if nbr.size == 0:
            nbr = np.zeros(1, np.uint32)
        return self.L.ref_csr_from_arrays(n, np.ascontiguousarray(in_offsets, np.uint64), nbr,
                                          np.ascontiguousarray(out_degree, np.uint32))

    def csr_rmat(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1):
        """The RMAT benchmark graph as a reference CsrGraph, built in place on
        all host threads (csr_inplace.hpp; the same arrays as build_csr)."""
        return self.L.ref_csr_rmat(scale, edge_factor, a, b, c, seed)

    def csr_arrays(self, h) -> CsrArrays:
        n = self.L.ref_csr_vertex_count(h)
        e = self.L.ref_csr_edge_count(h)
        d = self.L.ref_csr_dangling_count(h)
        off = np.zeros(n + 1, np.uint64)
        nbr = np.zeros(max(e, 1), np.uint32)
        deg = np.zeros(max(n, 1), np.uint32)
        dang = np.zeros(max(d, 1), np.uint32)
        self.L.ref_csr_copy(h, off, nbr, deg, dang)
        return CsrArrays(n, off, nbr[:e], deg[:n], dang[:d])

    def build_csr(self, n, pairs) -> CsrArrays:
        h = self.build_csr_handle(n, pairs)
        try:
            return self.csr_arrays(h)
        finally:
            self.free_csr(h)

    def pagerank(self, h, alpha=0.85, tol=1e-6, norm="l1", max_iter=500, trace=False,
                 want_ranks=True):
        n = self.L.ref_csr_vertex_count(h)
        ranks = np.zeros(max(n, 1), np.float64) if want_ranks else None
        it, conv, ms = C.c_int(), C.c_int(), C.c_double()
        tr = np.zeros(max_iter, np.float64) if trace else None
        st = self.L.ref_pagerank(h, alpha, tol, _norm_id(norm), max_iter,
                                 ranks.ctypes.data if want_ranks else None,
                                 C.byref(it), C.byref(conv),
                                 tr.ctypes.data if trace else None, C.byref(ms))
        if st == 1:
            raise ValueError("reference pagerank: invalid argument")
        if st != 0:
            raise RuntimeError("reference pagerank failed")
        out = dict(iterations=it.value, converged=bool(conv.value), elapsed_ms=ms.value)
        if want_ranks:
            out["ranks"] = ranks[:n]
        if trace:
            out["err_trace"] = tr[: it.value]
        return out

    def dense_pagerank(self, n, pairs, alpha, tol, norm, max_iter=500):
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
        if pairs.size == 0:
            pairs = np.zeros(2, np.uint32)
            m = 0
        else:
            m = pairs.size // 2
        ranks = np.zeros(n, np.float64)
        it, conv = C.c_int(), C.c_int()
        self.L.ref_dense_pagerank(n, pairs, m, alpha, tol, _norm_id(norm), max_iter, ranks,
                                  C.byref(it), C.byref(conv))
        return dict(ranks=ranks, iterations=it.value, converged=bool(conv.value))

    def error_norm(self, norm, r, s) -> float:
        r = np.ascontiguousarray(r, np.float64)
        s = np.ascontiguousarray(s, np.float64)
        st = C.c_int()
        v = self.L.ref_error_norm(_norm_id(norm), r.ctypes.data, s.ctypes.data, r.size, s.size,
                                  C.byref(st))
        if st.value:
            raise ValueError("error_norm: invalid argument")
        return v

    def estimate_iterations(self, alpha, tol) -> int:
        v = self.L.ref_estimate_iterations(alpha, tol)
        if v < 0:
            raise ValueError("estimate_iterations: argument outside (0, 1)")
        return v
