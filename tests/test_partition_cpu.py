"""CPU (gloo, world size 2): the multi-GPU exchange protocol of
paper_2108_02997_b200.distributed, restated on the host with numpy.

Each rank owns a contiguous, cost-balanced row range, pulls its rows from the
full previous contribution vector, then the ranks all-gather (a) their new
contribution rows and (b) their partial sums, and every rank reduces the
partials in rank order.  The run must reproduce the single-process oracle:
same iteration count, ranks within 1e-12."""
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
