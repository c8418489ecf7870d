"""Full-vector parity at benchmark size: the reference's own pagerank()
(oracle/_ref, the unmodified headers) run on the GPU box's host cores, one
thread per run, against the B200 path on the same graphs — every rank of
every run compared, not a sample (north_star bars: iterations exact, or +-1
only where the reference's err is within 1e-3 tau of tau; ranks Linf <= 1e-10).

  C2  RMAT-22 damping sweep: 11 alphas batched as lanes, tau 1e-6, L1
  C3  grid 4096^2: alpha .85 to tau 1e-10 under L1, L2 and Linf

The reference graphs are built independently of the GPU: C2 by the in-place
builder (oracle/csr_inplace.hpp, fingerprint-pinned to build_csr), C3 by the
reference's own build_csr from the oracle's grid generator."""
import threading

import numpy as np
import pytest

from conftest import load_golden

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RANK_TOL = 1e-10


def iterations_match(got, want, trace, tol):
    if got == want:
        return True
    t = min(got, want)
    return abs(got - want) == 1 and any(abs(trace[i] - tol) <= 1e-3 * tol for i in (t - 1, t) if i < len(trace))


def ref_runs(ref, h, jobs):
    """[(alpha, tol, norm)] -> reference results, all concurrently."""
    out = [None] * len(jobs)

    def work(i):
        a, tol, norm = jobs[i]
        out[i] = ref.pagerank(h, a, tol, norm, 500, trace=True)
    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return out


def test_c2_damping_sweep_full_vectors(prl, ref):
    gold = load_golden("c2_rmat22.json")
    alphas = [lane["alpha"] for lane in gold["lanes"]]
    h = ref.csr_rmat(22, 16, 0.57, 0.19, 0.19, gold["seed"])
    try:
        assert ref.L.ref_csr_edge_count(h) == gold["graph"]["e"]
        want = ref_runs(ref, h, [(a, 1e-6, "l1") for a in alphas])
    finally:
        ref.free_csr(h)
    g = prl.generate_rmat(22, 16, 0.57, 0.19, 0.19, gold["seed"])
    got = prl.pagerank_batched(g, alphas, 1e-6, prl.NormKind.L1, 500)
    for k, (r, w) in enumerate(zip(got.results, want)):
        assert iterations_match(r.iterations, w["iterations"], w["err_trace"], 1e-6), (alphas[k], r.iterations)
        assert r.converged == w["converged"]
        assert float(np.max(np.abs(r.ranks - w["ranks"]))) <= RANK_TOL, alphas[k]


def test_c3_grid_all_norms_full_vectors(prl, ref, oracle):
    gold = load_golden("c3_grid4096.json")
    n, pairs = oracle.grid(4096, 0.6, 0.01, gold["seed"])
    h = ref.build_csr_handle(n, pairs)
    del pairs
    try:
        want = ref_runs(ref, h, [(0.85, 1e-10, nm) for nm in ("l1", "l2", "linf")])
    finally:
        ref.free_csr(h)
    g = prl.generate_grid(4096, 0.6, 0.01, gold["seed"])
    kinds = (prl.NormKind.L1, prl.NormKind.L2, prl.NormKind.LInf)
    for kind, w in zip(kinds, want):
        r = prl.pagerank(g, prl.PageRankConfig(0.85, 1e-10, kind, 500))
        assert iterations_match(r.iterations, w["iterations"], w["err_trace"], 1e-10), (kind, r.iterations)
        assert float(np.max(np.abs(r.ranks - w["ranks"]))) <= RANK_TOL, kind
