"""GPU: the multi-GPU 1D-partition path (paper_2108_02997_b200.distributed).

Only one GPU is available per call, so partitions are emulated in one process
(same kernels, buffer copies instead of NCCL) and NCCL is exercised with a
world of 1.  Results must match the fused single-GPU run: identical iteration
counts and ranks within 1e-13 (only the cross-rank order of the partial sums
differs)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nranks", [1, 2, 3, 5])
@pytest.mark.parametrize("alphas", [[0.85], [0.5, 0.85, 1.0]])
def test_emulated_partitions_match_fused(prl, nranks, alphas):
    from paper_2108_02997_b200 import distributed
    g = prl.generate_rmat(14, 16, 0.57, 0.19, 0.19, 2108)
    want = prl.pagerank_batched(g, alphas, 1e-9)
    got = distributed.emulate(g, alphas, nranks, 1e-9)
    for k in range(len(alphas)):
        assert got.iterations[k] == want.results[k].iterations
        assert np.max(np.abs(got.ranks[k] - want.results[k].ranks)) <= 1e-13


def test_partition_plan_covers_rows_and_sources(prl):
    from paper_2108_02997_b200 import distributed
    g = prl.generate_rmat(16, 16, 0.57, 0.19, 0.19, 2108)
    p = distributed._Part(g, [0.85], 1e-6, prl.NormKind.L1, 500, 0, 0, 4, g.device)
    parts = p.parts
    assert parts[0].row_begin == 0 and parts[-1].row_end == g.vertex_count
    assert parts[0].src_begin == 0 and parts[-1].src_end == p.nsrc
    for a, b in zip(parts, parts[1:]):
        assert a.row_end == b.row_begin and a.src_end == b.src_begin and a.task_end == b.task_begin
    # cost balance: no rank holds more than ~2x the average edges
    off = g.in_offsets  # reference layout; edges per rank in engine order via the plan sizes
    assert all(q.row_end >= q.row_begin for q in parts)
    p.close()


def test_nccl_world_of_one(prl):
    import torch
    import torch.distributed as dist
    from paper_2108_02997_b200 import distributed
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29513")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = prl.generate_rmat(14, 16, 0.57, 0.19, 0.19, 2108)
        want = prl.pagerank_batched(g, [0.75, 0.85], 1e-8)
        got = distributed.run_distributed(g, [0.75, 0.85], 1e-8, want_ranks=True)
        for k in range(2):
            assert got.iterations[k] == want.results[k].iterations
            assert np.max(np.abs(got.ranks[k] - want.results[k].ranks)) <= 1e-13
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks", [1, 2, 3, 5])
@pytest.mark.parametrize("alphas", [[0.85], [0.5, 0.85, 1.0]])
def test_fused_peer_exchange_emulated(prl, nranks, alphas):
    """The peer-memory exchange: each rank's kernels store into the other
    ranks' buffers and count arrivals (ranks run one after another on this
    GPU, so nothing waits); must equal the fused single-GPU run."""
    from paper_2108_02997_b200 import distributed
    g = prl.generate_rmat(14, 16, 0.57, 0.19, 0.19, 2108)
    want = prl.pagerank_batched(g, alphas, 1e-9)
    got = distributed.emulate(g, alphas, nranks, 1e-9, fused=True)
    for k in range(len(alphas)):
        assert got.iterations[k] == want.results[k].iterations
        assert np.max(np.abs(got.ranks[k] - want.results[k].ranks)) <= 1e-13


def test_fused_exchange_sends_only_needed_rows(prl, monkeypatch):
    """Needed-only exchange: each rank stores fewer rows than 'every source row
    to every peer' (PRGPU_NEED=0), with identical results; one rank sends
    nothing."""
    from paper_2108_02997_b200 import distributed
    g = prl.generate_rmat(14, 16, 0.57, 0.19, 0.19, 2108)
    alphas = [0.5, 0.85, 1.0]
    assert distributed.emulate(g, alphas, 1, 1e-9, fused=True).sent_bytes == 0
    need = distributed.emulate(g, alphas, 3, 1e-9, fused=True)
    monkeypatch.setenv("PRGPU_NEED", "0")
    every = distributed.emulate(g, alphas, 3, 1e-9, fused=True)
    assert 0 < need.sent_bytes < every.sent_bytes
    assert np.array_equal(need.iterations, every.iterations)
    assert np.array_equal(need.ranks, every.ranks)


def test_fused_peer_graph_loop_single_rank(prl):
    """One rank, the whole loop as the CUDA graph prgpu_part_launch enqueues
    (the finalize kernel's arrival wait included)."""
    from paper_2108_02997_b200 import distributed
    g = prl.generate_rmat(14, 16, 0.57, 0.19, 0.19, 2108)
    want = prl.pagerank_batched(g, [0.6, 0.85], 1e-9)
    got = distributed.emulate(g, [0.6, 0.85], 1, 1e-9, fused=True, graph=True)
    for k in range(2):
        assert got.iterations[k] == want.results[k].iterations
        assert np.max(np.abs(got.ranks[k] - want.results[k].ranks)) <= 1e-13


def test_nccl_world_of_one_peer_exchange(prl):
    import torch
    import torch.distributed as dist
    from paper_2108_02997_b200 import distributed
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29514"
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = prl.generate_rmat(14, 16, 0.57, 0.19, 0.19, 2108)
        want = prl.pagerank_batched(g, [0.75, 0.85], 1e-8)
        got = distributed.run_distributed(g, [0.75, 0.85], 1e-8, want_ranks=True, exchange="peer")
        for k in range(2):
            assert got.iterations[k] == want.results[k].iterations
            assert np.max(np.abs(got.ranks[k] - want.results[k].ranks)) <= 1e-13
    finally:
        dist.destroy_process_group()


def test_fused_eight_ranks_eleven_lanes(prl):
    """The widest multi-GPU case: 8 ranks (the most one NVSwitch domain holds,
    every bit of the needed-rank mask), 11 damping lanes walking through all
    lane-width modes, dealt work; equal to the single-GPU run."""
    from paper_2108_02997_b200 import distributed
    g = prl.generate_rmat(16, 16, 0.57, 0.19, 0.19, 2108)
    alphas = [0.50, 0.55, 0.60, 0.65, 0.70, 0.75, 0.80, 0.85, 0.90, 0.95, 1.00]
    want = prl.pagerank_batched(g, alphas, 1e-8)
    got = distributed.emulate(g, alphas, 8, 1e-8, fused=True)
    assert got.sent_bytes > 0
    for k in range(len(alphas)):
        assert got.iterations[k] == want.results[k].iterations, k
        assert np.max(np.abs(got.ranks[k] - want.results[k].ranks)) <= 1e-13, k
