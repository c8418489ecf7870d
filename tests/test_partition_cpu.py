"""CPU (gloo, world size 2): the multi-GPU exchange protocol of
paper_2108_02997_b200.distributed, restated on the host with numpy.

Each rank owns a contiguous, cost-balanced row range, pulls its rows from the
full previous contribution vector, then the ranks all-gather (a) their new
contribution rows and (b) their partial sums, and every rank reduces the
partials in rank order.  The run must reproduce the single-process oracle:
same iteration count, ranks within 1e-12.  A second test restates the fused
peer-memory exchange (stores into every rank's buffers, parity-blocked
partials, arrival counters) with two processes over shared memory."""
import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

sys.path.insert(0, os.path.join(ROOT, "oracle"))


def split_rows(in_offsets, nranks):
    """Contiguous row ranges with equal cost (edges + 2 per row)."""
    n = in_offsets.size - 1
    cost = np.diff(in_offsets.astype(np.int64)) + 2
    pref = np.concatenate([[0], np.cumsum(cost)])
    bounds = [0] + [int(np.searchsorted(pref, pref[-1] * r / nranks)) for r in range(1, nranks)] + [n]
    return [(bounds[r], bounds[r + 1]) for r in range(nranks)]


def worker(rank, world, port, n, off, nbr, deg, alpha, tol, norm, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    lo, hi = split_rows(off, world)[rank]
    prev = np.full(n, 1.0 / n)
    dangling = deg == 0
    it, err = 0, np.inf
    while True:
        contrib = np.where(deg > 0, prev / np.maximum(deg, 1), 0.0)
        D_parts = torch.zeros(world, dtype=torch.float64)
        Dl = torch.tensor([float(np.sum(prev[lo:hi][dangling[lo:hi]]))], dtype=torch.float64)
        dist.all_gather_into_tensor(D_parts, Dl)
        D = 0.0
        for r in range(world):  # rank order
            D += float(D_parts[r])
        c0 = (1.0 - alpha) / n + alpha * D / n
        nxt = np.empty(hi - lo)
        for i, v in enumerate(range(lo, hi)):
            acc = 0.0
            for j in range(off[v], off[v + 1]):
                acc += contrib[nbr[j]]
            nxt[i] = c0 + alpha * acc
        d = nxt - prev[lo:hi]
        part = torch.tensor([np.sum(np.abs(d)), np.sum(d * d), np.max(np.abs(d)) if d.size else 0.0],
                            dtype=torch.float64)
        parts = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, part)
        l1 = l2 = linf = 0.0
        for p in parts:  # rank order: identical on every rank
            l1 += float(p[0]); l2 += float(p[1]); linf = max(linf, float(p[2]))
        err = [l1, np.sqrt(l2), linf][norm]
        # exchange the new rank rows (the GPU path exchanges contributions r/d)
        chunks = [None] * world
        dist.all_gather_object(chunks, nxt)
        prev = np.concatenate(chunks)
        it += 1
        if not (err >= tol and it < 500):
            break
    if rank == 0:
        out.put((it, prev))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("norm", [0, 1, 2])
def test_gloo_two_ranks_match_oracle(oracle, norm):
    n, pairs = oracle.rmat(9, 8, 0.57, 0.19, 0.19, 3)
    g = oracle.build_csr(n, pairs)
    h = oracle.build_csr_handle(n, pairs)
    want = oracle.pagerank(h, 0.85, 1e-9, norm)
    oracle.free_csr(h)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + norm
    procs = [ctx.Process(target=worker, args=(r, 2, port, n, g.in_offsets, g.in_neighbors,
                                              g.out_degree.astype(np.float64), 0.85, 1e-9, norm, q))
             for r in range(2)]
    for p in procs:
        p.start()
    it, ranks = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert it == want["iterations"]
    assert np.max(np.abs(ranks - want["ranks"])) <= 1e-12


def test_split_rows_balanced(oracle):
    n, pairs = oracle.rmat(12, 16, 0.57, 0.19, 0.19, 5)
    g = oracle.build_csr(n, pairs)
    parts = split_rows(g.in_offsets, 4)
    assert parts[0][0] == 0 and parts[-1][1] == n
    cost = np.diff(g.in_offsets.astype(np.int64)) + 2
    loads = [cost[a:b].sum() for a, b in parts]
    assert max(loads) <= 1.25 * (cost.sum() / 4) + cost.max()


def peer_worker(rank, world, names, n, off, nbr, deg, alpha, tol, out):
    """The fused peer-memory protocol of paper_2108_02997_b200 (pull.cuh,
    Params::fused) restated with processes and shared memory: a rank stores
    its new contribution rows and its partial vector straight into every
    rank's buffers (partials in slot [iteration parity][rank]), then bumps
    every rank's arrival counter; it reads the next iteration's inputs only
    after its own counter reaches world * (iteration + 1)."""
    import time
    from multiprocessing import shared_memory
    shm = {k: shared_memory.SharedMemory(name=v) for k, v in names.items()}
    contrib = [np.ndarray((2, n), np.float64, buffer=shm[f"c{r}"].buf) for r in range(world)]
    parts = [np.ndarray((2, world, 4), np.float64, buffer=shm[f"p{r}"].buf) for r in range(world)]
    arrive = np.ndarray((world,), np.int64, buffer=shm["a"].buf)
    locks = out["locks"]
    lo, hi = split_rows(off, world)[rank]
    dang = deg == 0
    prev = np.full(hi - lo, 1.0 / n)                 # this rank's rows only
    c0 = (1.0 - alpha) / n + alpha * (float(np.sum(dang)) / n) / n
    it = 0
    while True:
        par = it & 1
        c = contrib[rank][par]                       # every source's contribution, parity par
        nxt = np.empty(hi - lo)
        for i, v in enumerate(range(lo, hi)):
            nxt[i] = c0 + alpha * sum(c[nbr[j]] for j in range(off[v], off[v + 1]))
        d = nxt - prev
        mine = np.array([np.sum(np.abs(d)), np.sum(d * d), np.max(np.abs(d)) if d.size else 0.0,
                         float(np.sum(nxt[dang[lo:hi]]))])
        new_c = np.where(deg[lo:hi] > 0, nxt / np.maximum(deg[lo:hi], 1), 0.0)
        for r in range(world):                       # peer stores: rows and partials
            contrib[r][par ^ 1][lo:hi] = new_c
            parts[r][par][rank] = mine
        for r in range(world):                       # then arrive everywhere
            with locks[r]:
                arrive[r] += 1
        while arrive[rank] < world * (it + 1):       # the finalize kernel's wait
            time.sleep(0.0005)
        tot = np.zeros(4)
        for r in range(world):                       # rank order
            p = parts[rank][par][r]
            tot[0] += p[0]; tot[1] += p[1]; tot[2] = max(tot[2], p[2]); tot[3] += p[3]
        c0 = (1.0 - alpha) / n + alpha * tot[3] / n  # next teleport from the dangling sum
        prev = nxt
        it += 1
        if not (tot[0] >= tol and it < 500):
            break
    if rank == 0:
        out["q"].put(it)
    for s in shm.values():
        s.close()


def test_peer_exchange_protocol_two_processes(oracle):
    from multiprocessing import shared_memory
    ctx = mp.get_context("spawn")
    n, pairs = oracle.rmat(8, 8, 0.57, 0.19, 0.19, 11)
    g = oracle.build_csr(n, pairs)
    h = oracle.build_csr_handle(n, pairs)
    want = oracle.pagerank(h, 0.85, 1e-9, "l1")
    oracle.free_csr(h)
    world = 2
    deg = g.out_degree.astype(np.float64)
    shms = {}
    for r in range(world):
        shms[f"c{r}"] = shared_memory.SharedMemory(create=True, size=2 * n * 8)
        np.ndarray((2, n), np.float64, buffer=shms[f"c{r}"].buf)[0] = np.where(deg > 0, (1.0 / n) / np.maximum(deg, 1), 0)
        shms[f"p{r}"] = shared_memory.SharedMemory(create=True, size=2 * world * 4 * 8)
    shms["a"] = shared_memory.SharedMemory(create=True, size=world * 8)
    np.ndarray((world,), np.int64, buffer=shms["a"].buf)[:] = 0
    out = {"q": ctx.Queue(), "locks": [ctx.Lock() for _ in range(world)]}
    names = {k: v.name for k, v in shms.items()}
    procs = [ctx.Process(target=peer_worker, args=(r, world, names, n, g.in_offsets, g.in_neighbors,
                                                   deg, 0.85, 1e-9, out)) for r in range(world)]
    try:
        for p in procs:
            p.start()
        it = out["q"].get(timeout=300)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        assert it == want["iterations"]
    finally:
        for s in shms.values():
            s.close()
            s.unlink()
