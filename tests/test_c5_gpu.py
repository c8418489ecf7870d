"""C5 (BASELINE configs[4]): RMAT-28, 268M vertices, 4.26B edges, alpha sweep
{.95, .85, .75} batched K = 3, tau 1e-6, L2 norm — on one GPU.

A full reference run at this size takes hours and ~55 GB here, so
parity is checked one step at a time, which is size-independent: for every
lane, the GPU's last two iterates r_{t-1}, r_t (a run capped at t-1 iterations
reproduces the capped iterate bit for bit: runs are deterministic) are fed to
the oracle, which recomputes iteration t for a sample of rows exactly as
pagerank.hpp:85-93 does (dangling sum over the ascending dangling list, the
teleport, ascending-source sums of prev/out_degree) and the L2 norm of
r_t - r_{t-1} as norms.hpp:62-69 does (long double).  Bars: sampled rows
within Linf 1e-10 (north_star) and 1e-8 relative (measured: the rows differ
by one constant ~6e-19, the teleport term: the reference sums 169M dangling
ranks sequentially, the GPU as a tree, a ~3e-10 relative difference in D); the oracle's norm below
tau and equal to the GPU's reported err (1e-9 relative); the GPU's err trace
above tau at t-1; sum of ranks 1 +- 1e-9 (acceptance.cpp:134-161).
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ALPHAS = [0.95, 0.85, 0.75]
TOL = 1e-6


def test_c5_rmat28_k3_one_step_oracle(prl, oracle):
    g = prl.generate_rmat(28, 16, 0.57, 0.19, 0.19, 2108)
    n = g.vertex_count
    assert n == 1 << 28
    assert g.edge_count() > 4_000_000_000  # 64-bit row offsets in use
    deg = g.out_degree_only()
    assert int(np.count_nonzero(deg == 0)) == int(g.info.dangling_count)

    full = prl.pagerank_batched(g, ALPHAS, TOL, prl.NormKind.L2, 500)
    its = [r.iterations for r in full.results]
    assert all(r.converged for r in full.results)
    assert its == sorted(its, reverse=True)  # iterations monotone in alpha

    # rows: hubs (engine rows 0..31 are the largest in-degrees) plus a seeded sample
    perm = np.zeros(n, np.uint32)
    prl._lib.check(prl._lib.lib().prgpu_graph_permutation(g.handle, perm.ctypes.data), "perm")
    rng = np.random.default_rng(2108)
    rows = np.unique(np.concatenate([perm[:32], rng.integers(0, n, 4096).astype(np.uint32)]))
    del perm
    off, nbr = g.rows(rows)
    assert int(off[-1]) > 1_000_000  # the hubs bring millions of in-edges

    for k, a in enumerate(ALPHAS):
        t = its[k]
        nxt = full.results[k].ranks
        s = float(np.sum(nxt, dtype=np.longdouble))
        assert abs(s - 1.0) <= 1e-9, (a, s)
        capped = prl.pagerank_batched(g, ALPHAS, TOL, prl.NormKind.L2, t - 1)
        prev = capped.results[k].ranks
        assert capped.results[k].iterations == t - 1
        want, _ = oracle.step_rows(prev, deg, a, off, nbr)
        got = nxt[rows]
        diff = np.abs(got - want)
        assert float(diff.max()) <= 1e-10, (a, float(diff.max()))
        assert float(np.max(diff / want)) <= 1e-8, (a, float(np.max(diff / want)))
        err = oracle.error_norm("l2", nxt, prev)
        assert err < TOL, (a, err)
        assert abs(err - full.results[k].final_err) <= 1e-9 * err, (a, err, full.results[k].final_err)
        assert full.trace[t - 2, k, 1] >= TOL * (1 + 1e-3), (a, full.trace[t - 2, k, 1])
        del capped, prev


def test_c5_two_rank_fused_partition_matches_single_gpu(prl):
    """The multi-GPU path at the largest config: two ranks of the 1D
    partition, fused peer exchange with lane modes and needed-only rows,
    emulated on one GPU (the ranks run one after another, stores land in each
    other's buffers), against the single-GPU run: same iterations per lane,
    ranks within 1e-13 (only the rank-order reduction of the partials
    differs)."""
    from paper_2108_02997_b200 import distributed
    g = prl.generate_rmat(28, 16, 0.57, 0.19, 0.19, 2108)
    single = prl.pagerank_batched(g, ALPHAS, TOL, prl.NormKind.L2, 500)
    two = distributed.emulate(g, ALPHAS, 2, TOL, prl.NormKind.L2, 500, want_ranks=True, fused=True)
    assert two.sent_bytes > 0
    for k in range(len(ALPHAS)):
        assert two.iterations[k] == single.results[k].iterations, k
        assert float(np.max(np.abs(two.ranks[k] - single.results[k].ranks))) <= 1e-13, k
