"""Multi-GPU pull PageRank: 1D row partition, one process per GPU.

Each rank owns a contiguous, cost-balanced range of engine rows (a hub row is
never split across ranks) and so a contiguous range of source ids.  Per
iteration:

  1. ``prgpu_part_step``     — local pull over the rank's rows (sm_100a kernel)
  2. exchange                — every rank's new contribution rows and its
                               partial-sum vector reach every rank
                               (``torch.distributed`` over NCCL / NVLink)
  3. ``prgpu_part_finalize`` — the ranks' partial vectors are reduced in rank
                               order, so c0 and the stop decision are identical
                               on every rank (and deterministic)

The exchanged buffers are torch tensors handed to the engine, so NCCL moves
them in place; engine work is enqueued on torch's current stream.
``emulate`` runs the same protocol with several partitions in one process on
one GPU (buffer copies instead of NCCL) — that is how the partitioned path is
checked bit-for-bit against the single-GPU run when only one GPU is present.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib
from .pagerank_lab import CsrGraph, NormKind, _params


@dataclass
class PartResult:
    iterations: np.ndarray     # [K]
    ranks: Optional[np.ndarray]  # [K, n] original vertex ids (when gathered)
    run_iterations: int
    loop_ms: float
    sent_bytes: int = 0        # fused exchange: bytes this rank stores into peers per all-lanes iteration


class _Part:
    """One rank's engine session plus its exchange buffers (torch tensors)."""

    def __init__(self, g: CsrGraph, alphas, tolerance, norm, max_iterations, stop_mask, rank,
                 nranks, device, fused: bool = False):
        import torch
        self.torch = torch
        self.g = g
        self.K = len(alphas)
        self.rank, self.nranks = rank, nranks
        self.fused = fused
        p, self._keep = _params(list(alphas), tolerance, norm, max_iterations, stop_mask)
        self._p = p
        nc, npart = C.c_uint64(), C.c_uint64()
        check(lib().prgpu_part_buffer_sizes(g.handle, C.byref(p), nranks, C.byref(nc),
                                            C.byref(npart)), "part sizes")
        dev = torch.device("cuda", device)
        self.contrib = torch.empty(nc.value, dtype=torch.float64, device=dev)
        # fused exchange: partials double-buffered by iteration parity, plus
        # the arrival counter the peers increment
        self.partials = torch.zeros(npart.value * (2 if fused else 1), dtype=torch.float64, device=dev)
        self.arrive = torch.zeros(1, dtype=torch.int32, device=dev) if fused else None
        self._s = C.c_void_p()
        check(lib().prgpu_part_create(g.handle, C.byref(p), rank, nranks, self.contrib.data_ptr(),
                                      self.partials.data_ptr(), C.byref(self._s)), "part create")
        parts = (_lib.Partition * nranks)()
        check(lib().prgpu_part_plan(self._s, parts), "part plan")
        self.parts = [parts[i] for i in range(nranks)]
        ex = _lib.Exchange()
        check(lib().prgpu_part_exchange(self._s, C.byref(ex)), "part exchange")
        self.stride = ex.stride
        self.nsrc = ex.nsrc
        self.ppr = ex.partials_per_rank
        base = self.contrib.data_ptr()
        # views of the two parity buffers and of each rank's rows in them
        self.buf = [self.contrib[(ex.contrib[i] - base) // 8:(ex.contrib[i] - base) // 8 +
                                 self.nsrc * self.stride] for i in (0, 1)]
        self.slot = self.partials.view(-1, self.ppr)[:nranks]

    def chunk(self, parity, r):
        q = self.parts[r]
        return self.buf[parity][q.src_begin * self.stride:q.src_end * self.stride]

    def set_stream(self):
        s = self.torch.cuda.current_stream(self.contrib.device).cuda_stream
        if not s:
            raise RuntimeError("run inside `with torch.cuda.stream(...)`: the legacy default "
                               "stream cannot be shared with the engine")
        check(lib().prgpu_part_set_stream(self._s, C.c_void_p(s)), "part stream")

    def init(self):
        check(lib().prgpu_part_init(self._s), "part init")

    def set_peers(self, peer_contrib, peer_partials, peer_arrive):
        """Fused exchange: device pointers (ints) of the other ranks' buffers, rank order."""
        n = len(peer_contrib)
        arr = (C.c_void_p * max(n, 1))
        check(lib().prgpu_part_set_peers(self._s, n, arr(*peer_contrib), arr(*peer_partials),
                                         arr(*peer_arrive), C.c_void_p(self.arrive.data_ptr())), "set peers")

    def launch(self):
        check(lib().prgpu_part_launch(self._s), "part launch")

    def shard(self) -> bool:
        return self.g.shard_info()["nranks"] > 1

    def need_bits(self):
        """This rank's bit of the needed-only exchange mask (shard graphs:
        from its own rows), one byte per source, as a device tensor."""
        torch = self.torch
        bits = torch.zeros((self.nsrc + 3) // 4 * 4, dtype=torch.uint8, device=self.contrib.device)
        check(lib().prgpu_part_need_local(self._s, C.c_void_p(bits.data_ptr())), "need local")
        return bits

    def set_need(self, bits):
        check(lib().prgpu_part_set_need(self._s, C.c_void_p(bits.data_ptr())), "set need")

    def dealt(self) -> bool:
        """Work dealt round-robin (fused partitions): rows are not one range."""
        d = C.c_int()
        check(lib().prgpu_part_owned_ranks_device(self._s, None, 0, C.byref(d)), "owned ranks")
        return bool(d.value)

    def owned_ranks_into(self, out) -> None:
        """Add this rank's rows (every lane, engine row order) into the zeroed
        device tensor out[K][n]."""
        d = C.c_int()
        check(lib().prgpu_part_owned_ranks_device(self._s, C.c_void_p(out.data_ptr()), out.shape[1],
                                                  C.byref(d)), "owned ranks")

    def sent_bytes(self) -> int:
        """Bytes this rank stores into its peers per all-lanes iteration (fused)."""
        rows, rd = C.c_uint64(), C.c_uint32()
        check(lib().prgpu_part_sent_rows(self._s, C.byref(rows), C.byref(rd)), "sent rows")
        return int(rows.value) * int(rd.value) * 8

    def step(self) -> int:
        par = C.c_int()
        check(lib().prgpu_part_step(self._s, C.byref(par)), "part step")
        return par.value

    def finalize(self):
        check(lib().prgpu_part_finalize(self._s), "part finalize")

    def active(self) -> bool:
        a = C.c_int()
        check(lib().prgpu_part_active(self._s, C.byref(a)), "part active")
        return bool(a.value)

    def local_ranks(self, lane) -> np.ndarray:
        q = self.parts[self.rank]
        out = np.zeros(q.row_end - q.row_begin, np.float64)
        check(lib().prgpu_part_local_ranks(self._s, lane, out.ctypes.data), "local ranks")
        return out

    def close(self):
        if self._s:
            lib().prgpu_session_free(self._s)
            self._s = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _permutation(g: CsrGraph) -> np.ndarray:
    perm = np.zeros(g.vertex_count, np.uint32)
    check(lib().prgpu_graph_permutation(g.handle, perm.ctypes.data), "permutation")
    return perm


def _assemble(g: CsrGraph, chunks_by_rank, K) -> np.ndarray:
    """Concatenate per-rank engine-row chunks and map back to caller ids."""
    perm = _permutation(g)
    out = np.zeros((K, g.vertex_count), np.float64)
    for k in range(K):
        eng = np.concatenate([c[k] for c in chunks_by_rank])
        out[k, perm] = eng
    return out


def emulate(g: CsrGraph, alphas: Sequence[float], nranks: int, tolerance=1e-6,
            norm: NormKind = NormKind.L1, max_iterations: int = 500, stop_mask: int = 0,
            want_ranks: bool = True, fused: bool = False, graph: bool = False,
            shards: Optional[Sequence[CsrGraph]] = None) -> PartResult:
    """All `nranks` partitions in this process on this GPU.  Default: the
    exchange is a device copy of each rank's rows into every other rank's
    buffers (what NCCL does between GPUs).  fused=True: the ranks' kernels
    store into each other's buffers and count arrivals themselves (the
    peer-memory path); the ranks run one after another, so no kernel ever
    waits on another.  graph=True (one rank only): the fused loop as the
    CUDA graph prgpu_part_launch enqueues.  shards: the ranks' shard graphs
    (each holds its own rows' edges only)."""
    import torch
    if graph and (not fused or nranks != 1):
        raise ValueError("emulate: graph=True needs fused=True and nranks == 1 (ranks would wait on each other)")
    dev = g.device
    # shards: one shard graph per rank (generate_rmat(shard=(r, nranks))), g any of them
    parts = [_Part(shards[r] if shards else g, alphas, tolerance, norm, max_iterations, stop_mask, r, nranks, dev,
                   fused=fused) for r in range(nranks)]
    stream = torch.cuda.Stream(device=dev)  # a real stream: the legacy default is handle 0
    with torch.cuda.stream(stream):
        return _emulate_on(parts, alphas, max_iterations, want_ranks, g, fused, graph)


def _emulate_on(parts, alphas, max_iterations, want_ranks, g, fused=False, graph=False):
    import torch
    for p in parts:
        p.set_stream()
    if fused:
        if len(parts) > 1 and parts[0].shard():  # the ranks' bits summed (disjoint: = OR)
            total = sum(p.need_bits() for p in parts)
            for p in parts:
                p.set_need(total)
        for p in parts:
            peers = [q for q in parts if q is not p]
            p.set_peers([q.contrib.data_ptr() for q in peers], [q.partials.data_ptr() for q in peers],
                        [q.arrive.data_ptr() for q in peers])
    for p in parts:
        p.init()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    its = 0
    if graph:
        parts[0].launch()
        its = -1
    while 0 <= its < max_iterations:
        pars = [p.step() for p in parts]
        par = pars[0]
        if not fused:
            for dst in parts:
                for r, src in enumerate(parts):
                    if src is not dst:
                        dst.chunk(par, r).copy_(src.chunk(par, r))
                        dst.slot[r].copy_(src.slot[r])
        for p in parts:
            p.finalize()
        its += 1
        if not parts[0].active():
            break
    stop.record()
    torch.cuda.synchronize()
    K = len(alphas)
    res = PartResult(iterations=np.zeros(K, np.int32), ranks=None, run_iterations=0,
                     loop_ms=start.elapsed_time(stop))
    if want_ranks:
        if parts[0].dealt():  # disjoint owned rows summed over the ranks
            eng = torch.zeros((K, g.vertex_count), dtype=torch.float64, device=parts[0].contrib.device)
            for p in parts:
                p.owned_ranks_into(eng)
            res.ranks = _to_caller_host(eng, g, parts[0].contrib.device)
        else:
            chunks = [[p.local_ranks(k) for k in range(K)] for p in parts]
            res.ranks = _assemble(g, chunks, K)
    res.iterations[:] = _lane_iterations(parts[0])
    res.run_iterations = int(res.iterations.max())
    if fused:
        res.sent_bytes = max(p.sent_bytes() for p in parts)
    for p in parts:
        p.close()
    return res


def _lane_iterations(part: _Part) -> np.ndarray:
    """Per-lane iteration counts from the session's result call."""
    K = part.K
    its = np.zeros(K, np.int32)
    r = _lib.Result(None, its.ctypes.data_as(C.POINTER(C.c_int)), None, None, None, 0.0, 0)
    check(lib().prgpu_session_results(part._s, C.byref(r)), "results")
    return its


def run_distributed(g: CsrGraph, alphas: Sequence[float], tolerance=1e-6,
                    norm: NormKind = NormKind.L1, max_iterations: int = 500, stop_mask: int = 0,
                    want_ranks: bool = False, exchange: str = "nccl") -> PartResult:
    """One rank of an N-GPU run (torch.distributed initialised with NCCL,
    one process per GPU).

    exchange="nccl": one all-gather per iteration of every rank's new
    contribution rows and partial-sum vector, between host-enqueued pull and
    finalize kernels.  exchange="peer": the fused path — the ranks map each
    other's buffers (CUDA IPC), the pull kernel stores every contribution row
    and the partials straight into all peers over NVLink and the finalize
    kernel waits for the arrivals; the whole loop is one CUDA graph per rank,
    no collective call and no host round trip per iteration.
    exchange="peer-host": the same fused kernels and IPC mappings (peer
    stores, system-scope fences, arrival counters), but the host steps the
    loop: pull, stream sync, a barrier across ranks, then the finalize — whose
    arrival wait is already satisfied, so no kernel ever waits on another
    process.  Slower (a host round trip per iteration); it is what runs the
    fused exchange between processes that share one GPU (tests), where
    kernels spinning on each other are not allowed to co-run."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    stream = torch.cuda.Stream(device=g.device)  # engine, copies and NCCL share it
    with torch.cuda.stream(stream):
        if exchange in ("peer", "peer-host"):
            return _run_peer_on(g, alphas, tolerance, norm, max_iterations, stop_mask, want_ranks,
                                rank, world, host_steps=exchange == "peer-host")
        if exchange != "nccl":
            raise ValueError("exchange must be 'nccl', 'peer' or 'peer-host'")
        return _run_distributed_on(g, alphas, tolerance, norm, max_iterations, stop_mask, want_ranks,
                                   rank, world)


def _ipc_export(ptr: int):
    h = (C.c_char * 64)()
    off = C.c_uint64()
    check(lib().prgpu_ipc_export(C.c_void_p(ptr), h, C.byref(off)), "ipc export")
    return bytes(h), off.value


def _ipc_open(handle: bytes, offset: int, device: int) -> int:
    p = C.c_void_p()
    check(lib().prgpu_ipc_open((C.c_char * 64).from_buffer_copy(handle), offset, device, C.byref(p)),
          "ipc open")
    return p.value


def _agree_min(flag: int, device) -> int:
    """MIN of an int over the ranks, on whatever backend the group runs
    (NCCL wants a device tensor, gloo a host one)."""
    import torch
    import torch.distributed as dist
    on_host = dist.get_backend() == "gloo"
    t = torch.tensor([flag], dtype=torch.int32, device="cpu" if on_host else device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return int(t.item())


def _run_peer_on(g, alphas, tolerance, norm, max_iterations, stop_mask, want_ranks, rank, world,
                 host_steps: bool = False):
    import torch
    import torch.distributed as dist
    part = _Part(g, alphas, tolerance, norm, max_iterations, stop_mask, rank, world, g.device, fused=True)
    part.set_stream()
    opened = []  # (ptr, offset) to close
    peers = ([], [], [])
    ok = True
    try:
        mine = [_ipc_export(t.data_ptr()) for t in (part.contrib, part.partials, part.arrive)] if world > 1 else []
    except Exception:
        ok, mine = False, []
    table = [None] * world
    if world > 1:
        dist.all_gather_object(table, mine)
        ok = ok and all(t for t in table)
        for r in range(world):
            if r == rank or not ok:
                continue
            for j in range(3):
                try:
                    hnd, off = table[r][j]
                    ptr = _ipc_open(hnd, off, g.device)
                except Exception:
                    ok = False
                    break
                opened.append((ptr, off))
                peers[j].append(ptr)
        # every rank mapped every peer, or all fall back to the NCCL exchange
        if _agree_min(1 if ok else 0, part.contrib.device) == 0:
            for ptr, off in opened:
                lib().prgpu_ipc_close(C.c_void_p(ptr), off)
            part.close()
            return _run_distributed_on(g, alphas, tolerance, norm, max_iterations, stop_mask, want_ranks,
                                       rank, world)
    # set-up succeeded on EVERY rank, or all ranks release the mappings and
    # run the NCCL exchange together (a rank that failed alone would leave the
    # others spinning in the finalize wait on arrivals that never come)
    setup_ok = True
    try:
        if world > 1 and part.shard():  # the needed-only mask from every rank's rows
            bits = part.need_bits()
            if dist.get_backend() == "gloo":
                hb = bits.cpu()
                dist.all_reduce(hb, op=dist.ReduceOp.SUM)
                bits.copy_(hb)
            else:
                dist.all_reduce(bits, op=dist.ReduceOp.SUM)
            part.set_need(bits)
        part.set_peers(*peers)
        part.init()
        torch.cuda.current_stream(part.contrib.device).synchronize()
    except Exception:
        setup_ok = False
    if world > 1:
        setup_ok = _agree_min(1 if setup_ok else 0, part.contrib.device) == 1
    if not setup_ok:
        # nothing was launched: no peer stores can be in flight
        for ptr, off in opened:
            lib().prgpu_ipc_close(C.c_void_p(ptr), off)
        part.close()
        if world == 1:
            raise RuntimeError("fused exchange set-up failed on the only rank")
        return _run_distributed_on(g, alphas, tolerance, norm, max_iterations, stop_mask, want_ranks,
                                   rank, world)
    launched = False
    try:
        if world > 1:
            dist.barrier()  # every rank's counters are reset before anyone arrives
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        if host_steps:
            cur = torch.cuda.current_stream(part.contrib.device)
            launched = True
            for _ in range(max_iterations):
                part.step()       # stores rows + partials into the peers, then arrives
                cur.synchronize()
                if world > 1:
                    dist.barrier()  # every rank's stores and arrivals are complete
                part.finalize()   # arrival wait already satisfied: returns at once
                cur.synchronize()
                if not part.active():
                    break
        else:
            part.launch()
            launched = True
        stop.record()
        torch.cuda.current_stream(part.contrib.device).synchronize()
        K = len(alphas)
        lane_its = _lane_iterations(part)
        res = PartResult(iterations=lane_its, ranks=None, run_iterations=int(lane_its.max()),
                         loop_ms=start.elapsed_time(stop), sent_bytes=part.sent_bytes())
        if world > 1:
            dist.barrier()  # no peer still stores into our buffers
        if want_ranks:
            res.ranks = _gather_ranks(part, g, K, world)
    finally:
        # on the error path our own loop is drained first (it finished, or the
        # bounded arrival wait trapped); peers' stores into our buffers can
        # only target iterations our loop waited for, so none is in flight
        if launched:
            try:
                torch.cuda.current_stream(part.contrib.device).synchronize()
            except Exception:
                pass
        for ptr, off in opened:
            lib().prgpu_ipc_close(C.c_void_p(ptr), off)
        part.close()
    return res


def _run_distributed_on(g, alphas, tolerance, norm, max_iterations, stop_mask, want_ranks, rank, world):
    import torch
    import torch.distributed as dist
    part = _Part(g, alphas, tolerance, norm, max_iterations, stop_mask, rank, world, g.device)
    part.set_stream()
    part.init()
    dev = part.contrib.device
    # ONE all-gather per iteration: each rank's row of the exchange buffer is
    # its new contribution rows (its source range, padded to the longest
    # range) followed by its partial-sum vector; every rank then copies the
    # peers' rows into place on the device
    lens = [(q.src_end - q.src_begin) * part.stride for q in part.parts]
    span = max(lens) if lens else 0
    row = span + part.ppr
    on_host = dist.get_backend() == "gloo"
    send = torch.zeros(row, dtype=torch.float64, device=dev)
    recv = torch.zeros(world * row, dtype=torch.float64, device=dev)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    start.record()
    its = 0
    # the stop flag is read back every WINDOW iterations only: launches after
    # convergence are no-ops on the device (the pull and finalize kernels
    # exit when no lane is active; the exchange re-sends unchanged rows)
    WINDOW = 4
    while its < max_iterations:
        par = part.step()
        if world > 1:
            send[:lens[rank]].copy_(part.chunk(par, rank))
            send[span:].copy_(part.slot[rank])
            if on_host:  # gloo (processes sharing a GPU in the tests): the collective on host copies
                hr = recv.new_empty(recv.shape, device="cpu")
                dist.all_gather_into_tensor(hr, send.cpu())
                recv.copy_(hr)
            else:
                dist.all_gather_into_tensor(recv, send)
            for r in range(world):
                if r != rank:
                    base = r * row
                    part.chunk(par, r).copy_(recv[base:base + lens[r]])
                    part.slot[r].copy_(recv[base + span:base + row])
        part.finalize()
        its += 1
        if its % WINDOW == 0 and not part.active():
            break
    stop.record()
    torch.cuda.synchronize()
    K = len(alphas)
    lane_its = _lane_iterations(part)
    res = PartResult(iterations=lane_its, ranks=None, run_iterations=int(lane_its.max()),
                     loop_ms=start.elapsed_time(stop))
    if want_ranks:
        res.ranks = _gather_ranks(part, g, K, world)
    part.close()
    return res


def _gather_ranks(part: _Part, g: CsrGraph, K: int, world: int) -> np.ndarray:
    """Every rank's rows of every lane gathered on the devices (one
    all-gather), put back in caller order there, one copy to the host."""
    import torch
    import torch.distributed as dist
    dev = part.contrib.device
    if part.dealt():  # rows dealt round-robin: disjoint rows summed across ranks
        eng = torch.zeros((K, g.vertex_count), dtype=torch.float64, device=dev)
        part.owned_ranks_into(eng)
        if world > 1:
            if dist.get_backend() == "gloo":  # host reduction (exact: disjoint rows, zeros elsewhere)
                host = eng.cpu()
                dist.all_reduce(host, op=dist.ReduceOp.SUM)
                eng.copy_(host)
            else:
                dist.all_reduce(eng, op=dist.ReduceOp.SUM)
        return _to_caller_host(eng, g, dev)
    rows = [q.row_end - q.row_begin for q in part.parts]
    ld = max(rows)
    local = torch.empty((K, ld), dtype=torch.float64, device=dev)
    check(lib().prgpu_part_local_ranks_device(part._s, C.c_void_p(local.data_ptr()), ld), "local ranks")
    if world > 1:
        gathered = torch.empty((world, K, ld), dtype=torch.float64, device=dev)
        if dist.get_backend() == "gloo":
            hg = torch.empty((world * K, ld), dtype=torch.float64)  # gloo: chunks along dim 0
            dist.all_gather_into_tensor(hg, local.cpu())
            gathered.copy_(hg.view(world, K, ld))
        else:
            dist.all_gather_into_tensor(gathered, local)
    else:
        gathered = local.unsqueeze(0)
    eng = torch.cat([gathered[r, :, :rows[r]] for r in range(world)], dim=1)  # [K][n], engine rows
    return _to_caller_host(eng, g, dev)


def _to_caller_host(eng, g: CsrGraph, dev) -> np.ndarray:
    """[K][n] engine-row ranks -> caller vertex order, on the host."""
    import torch
    perm = torch.from_numpy(_permutation(g).astype(np.int64)).to(dev)
    out = torch.empty_like(eng)
    out[:, perm] = eng
    host = torch.empty(out.shape, dtype=torch.float64, pin_memory=True)
    host.copy_(out)
    torch.cuda.current_stream(dev).synchronize()
    return host.numpy()
