"""Python mirror of the reference's pagerank_lab API, backed by libprgpu.so.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/include/pagerank_lab/*.hpp); every compute call goes
through the C ABI of include/prgpu.h into the sm_100a kernels.  Host-only
pieces the reference also keeps on the host (MatrixMarket text parsing,
estimate_iterations, grids, CSV formatting) are restated here and marked so.

Exceptions: std::invalid_argument -> ValueError, std::runtime_error ->
RuntimeError, MtxParseError -> MtxParseError(RuntimeError) with .line().
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, Iterable, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib

# ---------------------------------------------------------------------------
# norms.hpp:18-40
# ---------------------------------------------------------------------------


class NormKind(IntEnum):
    L1 = 0
    L2 = 1
    LInf = 2


all_norms = (NormKind.L1, NormKind.L2, NormKind.LInf)


def norm_name(kind: NormKind) -> str:
    """norms.hpp:23-30."""
    return {NormKind.L1: "l1", NormKind.L2: "l2", NormKind.LInf: "linf"}.get(NormKind(kind), "?")


def parse_norm(token: str) -> Optional[NormKind]:
    """norms.hpp:33-40 — case-insensitive l1 | l2 | linf, else None."""
    return {"l1": NormKind.L1, "l2": NormKind.L2, "linf": NormKind.LInf}.get(token.lower())


def _as_f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def error_norm(kind: NormKind, r, s, device: Optional[int] = None) -> float:
    """norms.hpp:48-78, computed on the device (deterministic tree reduction)."""
    r, s = _as_f64(r), _as_f64(s)
    if r.size != s.size:
        raise ValueError(f"error_norm: vector lengths differ ({r.size} vs {s.size})")
    if r.size == 0:
        raise ValueError("error_norm: empty vectors")
    out = C.c_double()
    dev = _lib.default_device() if device is None else device
    check(lib().prgpu_error_norm(int(kind), r.ctypes.data, s.ctypes.data, r.size, dev,
                                 C.byref(out)), "error_norm")
    return out.value


# ---------------------------------------------------------------------------
# graph.hpp
# ---------------------------------------------------------------------------


class MtxParseError(RuntimeError):
    """graph.hpp:22-32 — a malformed MatrixMarket stream; line() is 1-based."""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self._line = line

    def line(self) -> int:
        return self._line


@dataclass
class EdgeList:
    """graph.hpp:36-39.  edges: (m, 2) uint32 array of (source, target)."""
    vertex_count: int = 0
    edges: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), np.uint32))

    def __post_init__(self):
        self.edges = np.ascontiguousarray(np.asarray(self.edges, dtype=np.uint32).reshape(-1, 2))


class CsrGraph:
    """graph.hpp:47-60 — immutable reverse CSR.

    The graph lives on the device (built there by build_csr); the host arrays
    in_offsets / in_neighbors / out_degree / dangling are downloaded lazily in
    the reference layout (bit-identical to the reference's build_csr)."""

    def __init__(self, handle: C.c_void_p, device: int):
        self._h = handle
        self.device = device
        info = _lib.GraphInfo()
        check(lib().prgpu_graph_get_info(handle, C.byref(info)), "graph info")
        self.info = info
        self.vertex_count = int(info.vertex_count)
        self._host = None
        self._lock = threading.Lock()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().prgpu_graph_free(h)
            except Exception:
                pass
            self._h = None

    def release(self) -> None:
        """Free the device graph now (host arrays already downloaded stay)."""
        self.__del__()

    @property
    def handle(self):
        return self._h

    def edge_count(self) -> int:
        return int(self.info.edge_count)

    def _download(self):
        with self._lock:
            if self._host is None:
                n, e, d = self.vertex_count, self.edge_count(), int(self.info.dangling_count)
                off = np.zeros(n + 1, np.uint64)
                nbr = np.zeros(max(e, 1), np.uint32)
                deg = np.zeros(n, np.uint32)
                dang = np.zeros(max(d, 1), np.uint32)
                check(lib().prgpu_graph_download(self._h, off.ctypes.data, nbr.ctypes.data,
                                                 deg.ctypes.data, dang.ctypes.data), "download")
                self._host = (off, nbr[:e], deg, dang[:d])
            return self._host

    @property
    def in_offsets(self) -> np.ndarray:
        return self._download()[0]

    @property
    def in_neighbors(self) -> np.ndarray:
        return self._download()[1]

    @property
    def out_degree(self) -> np.ndarray:
        return self._download()[2]

    @property
    def dangling(self) -> np.ndarray:
        return self._download()[3]

    def in_edges(self, v: int) -> np.ndarray:
        off = self.in_offsets
        return self.in_neighbors[int(off[v]):int(off[v + 1])]

    def out_degree_only(self) -> np.ndarray:
        """out_degree[n] without downloading the edge arrays."""
        if self._host is not None:
            return self._host[2]
        deg = np.zeros(self.vertex_count, np.uint32)
        check(lib().prgpu_graph_download(self._h, None, None, deg.ctypes.data, None), "download")
        return deg

    def shard_info(self) -> dict:
        """rank, nranks, engine rows [row_begin, row_end) and edges held
        (prgpu_graph_shard_info; a whole graph: 0, 1, all rows, all edges)."""
        r, nr, rb, re_, le = C.c_int(), C.c_int(), C.c_uint32(), C.c_uint32(), C.c_uint64()
        check(lib().prgpu_graph_shard_info(self._h, C.byref(r), C.byref(nr), C.byref(rb), C.byref(re_),
                                           C.byref(le)), "shard info")
        return dict(rank=r.value, nranks=nr.value, row_begin=rb.value, row_end=re_.value,
                    local_edges=le.value)

    def rows(self, rows):
        """(off[len(rows)+1], nbr): the in-neighbours of the given vertices,
        ascending per row as in in_neighbors, without downloading the whole
        graph (prgpu_graph_rows)."""
        r = np.ascontiguousarray(rows, np.uint32)
        off = np.zeros(len(r) + 1, np.uint64)
        total = C.c_uint64()
        check(lib().prgpu_graph_rows(self._h, r.ctypes.data, len(r), off.ctypes.data, None, 0,
                                     C.byref(total)), "graph rows")
        nbr = np.zeros(max(int(total.value), 1), np.uint32)
        check(lib().prgpu_graph_rows(self._h, r.ctypes.data, len(r), off.ctypes.data, nbr.ctypes.data,
                                     len(nbr), C.byref(total)), "graph rows")
        return off, nbr[:int(total.value)]


def _new_graph(fn, *args, device: Optional[int] = None) -> CsrGraph:
    dev = _lib.default_device() if device is None else device
    h = C.c_void_p()
    check(fn(*args, dev, C.byref(h)), fn.__name__)
    return CsrGraph(h, dev)


def build_csr(el: EdgeList, device: Optional[int] = None) -> CsrGraph:
    """graph.hpp:204-234 on the device: sort by (target, source), unique,
    count, scan, fill; self-loops kept, duplicates dropped."""
    # vertex_count 0 gives the empty graph (graph.hpp:204-234); pagerank()
    # then raises (pagerank.hpp:74)
    pairs = np.ascontiguousarray(el.edges, dtype=np.uint32)
    return _new_graph(lib().prgpu_graph_build, el.vertex_count,
                      pairs.ctypes.data if pairs.size else None, pairs.shape[0], device=device)


def csr_from_arrays(vertex_count: int, in_offsets, in_neighbors, out_degree,
                    device: Optional[int] = None) -> CsrGraph:
    """A device graph from reference-layout host arrays (validated on the device)."""
    off = np.ascontiguousarray(in_offsets, np.uint64)
    nbr = np.ascontiguousarray(in_neighbors, np.uint32)
    deg = np.ascontiguousarray(out_degree, np.uint32)
    if off.size != vertex_count + 1 or deg.size != vertex_count:
        raise ValueError("csr_from_arrays: array lengths do not match vertex_count")
    return _new_graph(lib().prgpu_graph_from_csr, vertex_count, off.ctypes.data,
                      nbr.ctypes.data if nbr.size else None, deg.ctypes.data, device=device)


def generate_rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
                  c: float = 0.19, seed: int = 2108, device: Optional[int] = None,
                  shard: Optional[tuple] = None) -> CsrGraph:
    """RMAT graph generated and built on the device.
    shard=(rank, nranks): only that rank's rows' in-edges (SURVEY 8e set-up;
    prgpu_graph_generate_rmat_shard) for a partitioned run."""
    if shard is not None:
        rank, nranks = shard
        return _new_graph(lib().prgpu_graph_generate_rmat_shard, scale, edge_factor, a, b, c, seed,
                          rank, nranks, device=device)
    return _new_graph(lib().prgpu_graph_generate_rmat, scale, edge_factor, a, b, c, seed,
                      device=device)


def generate_grid(side: int, p: float = 0.6, longrange_frac: float = 0.01, seed: int = 2108,
                  device: Optional[int] = None) -> CsrGraph:
    """Road-like grid graph generated and built on the device."""
    return _new_graph(lib().prgpu_graph_generate_grid, side, p, longrange_frac, seed,
                      device=device)


# ---- MatrixMarket (graph.hpp:111-199, 238-251): the library's parallel parser ----

def _mtx_pairs(call) -> EdgeList:
    """Runs prgpu_mtx_parse / prgpu_mtx_load (`call` gets the output refs) and
    turns the result into an EdgeList; PRGPU_EPARSE comes back as
    (line, message)."""
    n, m, line = C.c_uint32(), C.c_uint64(), C.c_uint64()
    pairs = C.POINTER(C.c_uint32)()
    st = call(C.byref(n), C.byref(pairs), C.byref(m), C.byref(line))
    if st != _lib.PRGPU_OK:
        msg = lib().prgpu_last_error().decode(errors="replace")
        return st, int(line.value), msg
    try:
        arr = np.ctypeslib.as_array(pairs, shape=(2 * int(m.value),)).copy() if m.value else \
            np.zeros(0, np.uint32)
    finally:
        lib().prgpu_pairs_free(pairs)
    return EdgeList(int(n.value), arr.reshape(-1, 2))


def parse_matrix_market(text) -> EdgeList:
    """graph.hpp:111-199: coordinate pattern|real|integer, general|symmetric;
    MtxParseError(line) on malformed input.  Parsed by the library's
    multi-threaded host parser (prgpu_mtx_parse)."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    r = _mtx_pairs(lambda *out: lib().prgpu_mtx_parse(data, len(data), 0, *out))
    if isinstance(r, EdgeList):
        return r
    st, line, msg = r
    if st == _lib.PRGPU_EPARSE:
        prefix = f"line {line}: "
        raise MtxParseError(line, msg[len(prefix):] if msg.startswith(prefix) else msg)
    _lib.check(st, "parse_matrix_market")


def load_matrix_market(path) -> EdgeList:
    """graph.hpp:238-247 — errors name the file (std::runtime_error)."""
    path = os.fspath(path)
    r = _mtx_pairs(lambda *out: lib().prgpu_mtx_load(path.encode(), 0, *out))
    if isinstance(r, EdgeList):
        return r
    st, _, msg = r
    if st in (_lib.PRGPU_EPARSE, _lib.PRGPU_EIO):
        raise RuntimeError(msg)
    _lib.check(st, "load_matrix_market")


def load_csr_graph(path, device: Optional[int] = None) -> CsrGraph:
    """graph.hpp:249-251: parallel parse, then build_csr on the device
    (prgpu_graph_load_mtx)."""
    path = os.fspath(path)
    dev = _lib.default_device() if device is None else device
    h = C.c_void_p()
    st = lib().prgpu_graph_load_mtx(path.encode(), 0, dev, C.byref(h), None)
    if st in (_lib.PRGPU_EPARSE, _lib.PRGPU_EIO):
        raise RuntimeError(lib().prgpu_last_error().decode(errors="replace"))
    check(st, "load_csr_graph")
    return CsrGraph(h, dev)


# ---------------------------------------------------------------------------
# pagerank.hpp
# ---------------------------------------------------------------------------


@dataclass
class PageRankConfig:
    """pagerank.hpp:23-40."""
    alpha: float = 0.85
    tolerance: float = 1e-6
    norm: NormKind = NormKind.L1
    max_iterations: int = 500

    def validate(self) -> None:
        if not (self.alpha >= 0.0 and self.alpha <= 1.0):
            raise ValueError(f"alpha must be in [0, 1], got {self.alpha}")
        if not (self.tolerance > 0.0):
            raise ValueError(f"tolerance must be positive, got {self.tolerance}")
        if self.max_iterations < 1:
            raise ValueError(f"max_iterations must be >= 1, got {self.max_iterations}")


@dataclass
class PageRankResult:
    """pagerank.hpp:42-47; `elapsed` is the device loop time in ms."""
    ranks: np.ndarray
    iterations: int = 0
    converged: bool = False
    elapsed: float = 0.0
    final_err: float = math.inf


IterationObserver = Callable[[int, np.ndarray, float], None]


@dataclass
class BatchedRun:
    """K lanes run together: per-lane results plus the per-iteration norm trace."""
    results: list
    trace: np.ndarray        # [iterations_run, K, 4]: L1, L2, LInf, L1-vs-ref
    loop_ms: float
    run_iterations: int


def _params(alphas: Sequence[float], tolerance, norm: NormKind, max_iterations: int,
            stop_mask: int = 0, ref: Optional[np.ndarray] = None):
    K = len(alphas)
    a = (C.c_double * K)(*alphas)
    tols = None
    tol = tolerance
    if isinstance(tolerance, (list, tuple, np.ndarray)):
        tols = (C.c_double * K)(*tolerance)
        tol = float(tolerance[0])
    p = _lib.Params(K, a, tols, float(tol), int(norm), stop_mask, int(max_iterations),
                    ref.ctypes.data_as(C.POINTER(C.c_double)) if ref is not None else None)
    return p, (a, tols, ref)  # keep the buffers alive


def pagerank_batched(g: CsrGraph, alphas: Sequence[float], tolerance=1e-6,
                     norm: NormKind = NormKind.L1, max_iterations: int = 500,
                     stop_mask: int = 0, ref_ranks=None, want_ranks: bool = True,
                     series: bool = False) -> BatchedRun:
    """K = len(alphas) PageRank runs that share every edge visit (BASELINE C2).

    series=True: the same results from one alpha = 1 chain and per-lane
    weighted sums (prgpu_pagerank_series): one pull per iteration of the
    slowest lane instead of one per lane-iteration."""
    K = len(alphas)
    if not 1 <= K <= _lib.MAX_LANES:
        raise ValueError(f"pagerank_batched: 1..{_lib.MAX_LANES} alphas per run")
    for a in alphas:
        PageRankConfig(alpha=a, tolerance=float(np.min(tolerance)), norm=norm,
                       max_iterations=max_iterations).validate()
    n = g.vertex_count
    ref = _as_f64(ref_ranks) if ref_ranks is not None else None
    if ref is not None and ref.size != n:
        raise ValueError("ref_ranks length differs from vertex_count")
    p, keep = _params(list(alphas), tolerance, norm, max_iterations, stop_mask, ref)
    ranks = np.zeros((K, n), np.float64) if want_ranks else None
    its = np.zeros(K, np.int32)
    conv = np.zeros(K, np.uint8)
    ferr = np.zeros(K, np.float64)
    trace = np.zeros((max_iterations, K, 4), np.float64)
    r = _lib.Result(ranks.ctypes.data_as(C.POINTER(C.c_double)) if want_ranks else None,
                    its.ctypes.data_as(C.POINTER(C.c_int)),
                    conv.ctypes.data_as(C.POINTER(C.c_uint8)),
                    ferr.ctypes.data_as(C.POINTER(C.c_double)),
                    trace.ctypes.data_as(C.POINTER(C.c_double)), 0.0, 0)
    if series:
        if ref is not None:
            raise ValueError("pagerank_batched(series=True): ref_ranks not supported")
        check(lib().prgpu_pagerank_series(g.handle, C.byref(p), C.byref(r)), "pagerank_series")
    else:
        check(lib().prgpu_pagerank(g.handle, C.byref(p), C.byref(r)), "pagerank")
    del keep
    results = [PageRankResult(ranks[k] if want_ranks else None, int(its[k]), bool(conv[k]),
                              r.loop_ms, float(ferr[k])) for k in range(K)]
    return BatchedRun(results, trace[: r.run_iterations], r.loop_ms, r.run_iterations)


def pagerank(g: CsrGraph, cfg: PageRankConfig = PageRankConfig(),
             on_iteration: Optional[IterationObserver] = None) -> PageRankResult:
    """pagerank.hpp:70-108 on the device."""
    cfg.validate()
    if g.vertex_count == 0:
        raise ValueError("pagerank: graph has no vertices")
    if on_iteration is None:
        return pagerank_batched(g, [cfg.alpha], cfg.tolerance, cfg.norm,
                                cfg.max_iterations).results[0]
    n = g.vertex_count
    p, keep = _params([cfg.alpha], cfg.tolerance, cfg.norm, cfg.max_iterations)
    ranks = np.zeros(n, np.float64)
    its = np.zeros(1, np.int32)
    conv = np.zeros(1, np.uint8)
    ferr = np.zeros(1, np.float64)
    errors = []

    def cb(it, lane, rp, nn, err, user):
        arr = np.ctypeslib.as_array(rp, shape=(nn,))
        try:
            on_iteration(it, arr, err)
        except Exception as e:  # re-raised after the C call returns
            errors.append(e)

    cfun = _lib.OBSERVER(cb)
    r = _lib.Result(ranks.ctypes.data_as(C.POINTER(C.c_double)),
                    its.ctypes.data_as(C.POINTER(C.c_int)),
                    conv.ctypes.data_as(C.POINTER(C.c_uint8)),
                    ferr.ctypes.data_as(C.POINTER(C.c_double)), None, 0.0, 0)
    check(lib().prgpu_pagerank_observed(g.handle, C.byref(p), C.byref(r), cfun, None),
          "pagerank")
    del keep
    if errors:
        raise errors[0]
    return PageRankResult(ranks, int(its[0]), bool(conv[0]), r.loop_ms, float(ferr[0]))


def estimate_iterations(alpha: float, tolerance: float) -> int:
    """pagerank.hpp:113-123 (host scalar helper, as in the reference)."""
    if not (alpha > 0.0 and alpha < 1.0):
        raise ValueError(f"estimate_iterations: alpha must be in (0, 1), got {alpha}")
    if not (tolerance > 0.0 and tolerance < 1.0):
        raise ValueError(f"estimate_iterations: tolerance must be in (0, 1), got {tolerance}")
    q = math.log10(tolerance) / math.log10(alpha)
    est = int(math.floor(abs(q) + 0.5)) * (1 if q >= 0 else -1)  # std::lround
    return max(1, est)


def reference_config() -> PageRankConfig:
    """pagerank.hpp:126-128."""
    return PageRankConfig(0.85, 1e-6, NormKind.L1, 500)


def reference_ranks(g: CsrGraph) -> np.ndarray:
    """pagerank.hpp:130-132."""
    return pagerank(g, reference_config()).ranks


def reference_error(g: CsrGraph, ranks) -> float:
    """pagerank.hpp:135-138."""
    return error_norm(NormKind.L1, ranks, reference_ranks(g), device=g.device)


# ---------------------------------------------------------------------------
# csv.hpp (host formatting) and sweep.hpp
# ---------------------------------------------------------------------------


def format_double(x: float) -> str:
    """csv.hpp:17-21 — std::to_chars shortest round-trip: the shorter of the
    fixed and scientific forms of the shortest digits (ties: fixed)."""
    x = float(x)
    if math.isnan(x):
        return "nan" if math.copysign(1, x) > 0 else "-nan"
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    if x == 0:
        return "-0" if math.copysign(1, x) < 0 else "0"
    sign = "-" if x < 0 else ""
    r = repr(abs(x))
    mant, _, exp = r.partition("e")
    exp = int(exp) if exp else 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    if fp == "0":
        fp = ""
    digits = (ip + fp).lstrip("0")
    # decimal exponent of the first significant digit
    if ip.strip("0"):
        e10 = len(ip.lstrip("0")) - 1 + exp
    else:
        e10 = -(len(fp) - len(fp.lstrip("0"))) - 1 + exp
    digits = digits.rstrip("0") or "0"
    nd = len(digits)
    # scientific
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + "e" + ("-" if e10 < 0 else "+") + \
        f"{abs(e10):02d}"
    # fixed
    if e10 >= nd - 1:
        fixed = digits + "0" * (e10 - nd + 1)
    elif e10 >= 0:
        fixed = digits[: e10 + 1] + "." + digits[e10 + 1:]
    else:
        fixed = "0." + "0" * (-e10 - 1) + digits
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def csv_escape(field_: str) -> str:
    """csv.hpp:31-41."""
    if not any(ch in field_ for ch in ',"\n'):
        return field_
    return '"' + field_.replace('"', '""') + '"'


@dataclass
class SweepPlan:
    """sweep.hpp:31-56.  `fuse` (not in the reference) runs all alphas of a
    graph as one batched device run and derives every (tau, norm) cell from
    the per-iteration norm trace; fuse=False runs each cell separately
    exactly like the reference."""
    graphs: list = field(default_factory=list)
    alphas: list = field(default_factory=lambda: [0.85])
    tolerances: list = field(default_factory=lambda: [1e-6])
    norms: list = field(default_factory=lambda: [NormKind.L1])
    repeats: int = 5
    max_iterations: int = 500
    fuse: bool = True

    def validate(self) -> None:
        if not self.graphs:
            raise ValueError("sweep: no graphs")
        if not self.alphas:
            raise ValueError("sweep: no alphas")
        if not self.tolerances:
            raise ValueError("sweep: no tolerances")
        if not self.norms:
            raise ValueError("sweep: no norms")
        if self.repeats < 1:
            raise ValueError("sweep: repeats must be >= 1")
        if self.max_iterations < 1:
            raise ValueError("sweep: max_iterations must be >= 1")
        for a in self.alphas:
            if not (a >= 0.0 and a <= 1.0):
                raise ValueError(f"sweep: alpha out of [0, 1]: {a}")
        for t in self.tolerances:
            if not (t > 0.0):
                raise ValueError(f"sweep: tolerance must be positive: {t}")


@dataclass
class SweepRecord:
    """sweep.hpp:59-70."""
    graph: str = ""
    vertices: int = 0
    edges: int = 0
    alpha: float = 0.0
    tolerance: float = 0.0
    norm: NormKind = NormKind.L1
    iterations: int = 0
    converged: bool = False
    time_ms: float = 0.0
    err_vs_ref: float = 0.0


sweep_csv_header = "graph,vertices,edges,alpha,tolerance,norm,iterations,converged,time_ms,err_vs_ref"


def sweep_csv_row(r: SweepRecord) -> str:
    """sweep.hpp:75-96."""
    return ",".join([csv_escape(r.graph), str(r.vertices), str(r.edges), format_double(r.alpha),
                     format_double(r.tolerance), norm_name(r.norm), str(r.iterations),
                     "true" if r.converged else "false", format_double(r.time_ms),
                     format_double(r.err_vs_ref)])


def write_sweep_csv(os_, records: Iterable[SweepRecord]) -> None:
    os_.write(sweep_csv_header + "\n")
    for r in records:
        os_.write(sweep_csv_row(r) + "\n")


def default_damping_grid() -> list:
    """sweep.hpp:105-108."""
    return [0.50, 0.55, 0.60, 0.65, 0.70, 0.75, 0.80, 0.85, 0.90, 0.95, 1.00]


def default_tolerance_grid() -> list:
    """sweep.hpp:110-114."""
    return [1e0, 5e-1, 1e-1, 5e-2, 1e-2, 5e-3, 1e-3, 5e-4, 1e-4, 5e-5, 1e-5,
            5e-6, 1e-6, 5e-7, 1e-7, 5e-8, 1e-8, 5e-9, 1e-9, 5e-10, 1e-10]


def _graph_label(path) -> str:
    return os.path.splitext(os.path.basename(os.fspath(path)))[0]


def _cells_from_trace(trace_k: np.ndarray, iters_k: int, norm: NormKind, tol: float,
                      max_iter: int):
    """First iteration t (1-based) whose error under `norm` is < tol."""
    errs = trace_k[:iters_k, int(norm)]
    below = np.nonzero(errs < tol)[0]
    if below.size:
        t = int(below[0]) + 1
        return t, True
    return min(iters_k, max_iter), False


def run_sweep(plan: SweepPlan, log=None, graphs_override: Optional[dict] = None) -> list:
    """sweep.hpp:146-243.  Records come back sorted by (graph, norm, alpha,
    tolerance descending); iteration counts must agree across repeats.
    graphs_override maps a plan.graphs entry to a prebuilt CsrGraph."""
    plan.validate()
    records = []
    for path in plan.graphs:
        g = (graphs_override or {}).get(path)
        if g is None:
            g = load_csr_graph(path)
        label = _graph_label(path) if isinstance(path, (str, os.PathLike)) else str(path)
        ref = reference_ranks(g)  # untimed; doubles as the warm-up (sweep.hpp:160-161)
        recs = _sweep_fused(plan, g, label, ref) if plan.fuse else _sweep_cells(plan, g, label, ref)
        for rec in recs:
            if log is not None:
                log.write(sweep_csv_row(rec) + "\n")
        records.extend(recs)
    records.sort(key=lambda r: (r.graph, int(r.norm), r.alpha, -r.tolerance))
    return records


def _sweep_cells(plan: SweepPlan, g: CsrGraph, label: str, ref: np.ndarray) -> list:
    out = []
    for norm in plan.norms:
        for alpha in plan.alphas:
            for tol in plan.tolerances:
                cfg = PageRankConfig(alpha, tol, NormKind(norm), plan.max_iterations)
                total, result = 0.0, None
                for rep in range(plan.repeats):
                    r = pagerank(g, cfg)
                    total += r.elapsed
                    if rep > 0 and r.iterations != result.iterations:
                        raise RuntimeError(f"sweep: iteration count changed between repeats on {label}")
                    result = r
                out.append(SweepRecord(label, g.vertex_count, g.edge_count(), alpha, tol,
                                       NormKind(norm), result.iterations, result.converged,
                                       total / plan.repeats,
                                       error_norm(NormKind.L1, result.ranks, ref, device=g.device)))
    return out


def _sweep_fused(plan: SweepPlan, g: CsrGraph, label: str, ref: np.ndarray) -> list:
    """All alphas in batched lanes; every (tau, norm) cell read off the trace.

    time_ms of a cell = (batched loop time / iterations run) x the cell's
    iterations: the per-iteration cost of the fused run, charged per cell."""
    mask = 0
    for nm in plan.norms:
        mask |= 1 << int(nm)
    tau_min = float(min(plan.tolerances))
    out = []
    alphas = list(plan.alphas)
    for c0 in range(0, len(alphas), _lib.MAX_LANES):
        chunk = alphas[c0:c0 + _lib.MAX_LANES]
        runs = []
        for rep in range(plan.repeats):
            br = pagerank_batched(g, chunk, tau_min, NormKind(plan.norms[0]), plan.max_iterations,
                                  stop_mask=mask, ref_ranks=ref, want_ranks=False)
            if runs and not np.array_equal(br.trace, runs[0].trace, equal_nan=True):
                raise RuntimeError(f"sweep: iteration trace changed between repeats on {label}")
            runs.append(br)
        per_iter = sum(r.loop_ms for r in runs) / len(runs) / max(1, runs[0].run_iterations)
        br = runs[0]
        for norm in plan.norms:
            for k, alpha in enumerate(chunk):
                iters_k = br.results[k].iterations
                for tol in plan.tolerances:
                    t, conv = _cells_from_trace(br.trace[:, k, :], iters_k, NormKind(norm), tol,
                                                plan.max_iterations)
                    out.append(SweepRecord(label, g.vertex_count, g.edge_count(), alpha, tol,
                                           NormKind(norm), t, conv, per_iter * t,
                                           float(br.trace[t - 1, k, 3])))
    return out


@dataclass
class SensitivityFinding:
    """sweep.hpp:246-256."""
    graph: str = ""
    norm: NormKind = NormKind.L1
    first_failing_tolerance: Optional[float] = None
    single_iteration_tolerances: list = field(default_factory=list)


def detect_sensitivity(records: Sequence[SweepRecord]) -> list:
    """sweep.hpp:262-310 (host post-processing)."""
    if not records:
        raise ValueError("detect_sensitivity: no records")
    groups: dict = {}
    grid = sorted({r.tolerance for r in records}, reverse=True)
    for r in records:
        groups.setdefault((r.graph, int(r.norm)), []).append(r)
    report = []
    for key in sorted(groups):
        cells = sorted(groups[key], key=lambda r: -r.tolerance)
        name = f"{key[0]}/{norm_name(NormKind(key[1]))}"
        if len(cells) != len(grid):
            raise ValueError(f"detect_sensitivity: tolerance grid for {name} has gaps or duplicate cells")
        if any(c.tolerance != t for c, t in zip(cells, grid)):
            raise ValueError(f"detect_sensitivity: tolerance grid for {name} has gaps")
        f = SensitivityFinding(key[0], NormKind(key[1]))
        tail = len(cells)
        while tail > 0 and not cells[tail - 1].converged:
            tail -= 1
        if tail < len(cells):
            f.first_failing_tolerance = cells[tail].tolerance
        f.single_iteration_tolerances = [c.tolerance for c in cells if c.iterations == 1]
        report.append(f)
    return report


# ---------------------------------------------------------------------------
# device sessions (bench / repeated runs)
# ---------------------------------------------------------------------------


class Session:
    """A reusable device run: state and the CUDA graph (WHILE node) are built
    once; run() re-initialises ranks on the device and iterates to convergence."""

    def __init__(self, g: CsrGraph, alphas: Sequence[float], tolerance=1e-6,
                 norm: NormKind = NormKind.L1, max_iterations: int = 500, stop_mask: int = 0):
        self.g = g
        self.K = len(alphas)
        self.max_iterations = max_iterations
        p, self._keep = _params(list(alphas), tolerance, norm, max_iterations, stop_mask)
        self._p = p
        self._s = C.c_void_p()
        check(lib().prgpu_session_create(g.handle, C.byref(p), C.byref(self._s)), "session")

    def run(self) -> float:
        ms = C.c_double()
        check(lib().prgpu_session_run(self._s, C.byref(ms)), "session run")
        return ms.value

    def results(self, want_ranks: bool = False):
        n, K = self.g.vertex_count, self.K
        ranks = np.zeros((K, n), np.float64) if want_ranks else None
        its = np.zeros(K, np.int32)
        conv = np.zeros(K, np.uint8)
        ferr = np.zeros(K, np.float64)
        trace = np.zeros((self.max_iterations, K, 4), np.float64)
        r = _lib.Result(ranks.ctypes.data_as(C.POINTER(C.c_double)) if want_ranks else None,
                        its.ctypes.data_as(C.POINTER(C.c_int)),
                        conv.ctypes.data_as(C.POINTER(C.c_uint8)),
                        ferr.ctypes.data_as(C.POINTER(C.c_double)),
                        trace.ctypes.data_as(C.POINTER(C.c_double)), 0.0, 0)
        check(lib().prgpu_session_results(self._s, C.byref(r)), "session results")
        return dict(ranks=ranks, iterations=its, converged=conv.astype(bool), final_err=ferr,
                    trace=trace[: r.run_iterations], loop_ms=r.loop_ms,
                    run_iterations=r.run_iterations)

    def kernel_times(self) -> np.ndarray:
        """The last run's per-iteration pull-kernel time (ms) measured inside
        the CUDA graph (prgpu_session_kernel_times)."""
        buf = np.zeros(4096, np.float64)
        n = C.c_int()
        check(lib().prgpu_session_kernel_times(self._s, buf.ctypes.data_as(C.POINTER(C.c_double)), buf.size,
                                               C.byref(n)), "kernel times")
        return buf[: n.value].copy()

    def time_pull(self, launches: int) -> float:
        ms = C.c_double()
        check(lib().prgpu_session_time_pull(self._s, launches, C.byref(ms)), "time_pull")
        return ms.value

    def close(self):
        if self._s:
            lib().prgpu_session_free(self._s)
            self._s = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
