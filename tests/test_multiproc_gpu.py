"""The fused multi-GPU exchange between two real processes.

Two processes share cuda:0 (only one GPU per call here).  Each opens the
other's contribution buffers, rank-partial buffers and arrival counter by
CUDA IPC, and its pull kernel stores contribution rows and partials into the
peer and arrives there (system-scope fences, atomicAdd_system) — the
multi-GPU data path, across processes.  The loop is host-stepped
(exchange="peer-host": pull, sync, barrier, finalize), so no kernel ever spins
on the other process's kernel: kernels that wait on each other must not
share a GPU (B200_PROFILING.md; Xid 109).  Result: the same per-lane
iterations as the single-GPU run and ranks within 1e-13 (only the rank-order
reduction of the partials differs)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

ALPHAS = [0.95, 0.85, 0.5]


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("scale,exchange", [(14, "peer-host"), (18, "peer-host"), (16, "nccl")])
def test_two_processes_fused_exchange_match_single_gpu(prl, tmp_path, scale, exchange):
    """exchange="nccl" runs the collective path (one all-gather per
    iteration; on gloo here, as the processes share a GPU)."""
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(r), WORLD_SIZE="2",
                   LOCAL_RANK="0")
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mp_worker.py"),
                                       str(tmp_path / f"r{r}.npz"), str(scale), ",".join(map(str, ALPHAS)),
                                       exchange],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=600)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-4000:]
    g = prl.generate_rmat(scale, 16, 0.57, 0.19, 0.19, 2108)
    single = prl.pagerank_batched(g, ALPHAS, 1e-9, prl.NormKind.L1, 200)
    for r in range(2):
        d = np.load(tmp_path / f"r{r}.npz")
        if exchange != "nccl":
            assert int(d["sent"]) > 0  # rows really crossed to the peer
        for k, res in enumerate(single.results):
            assert int(d["iterations"][k]) == res.iterations, (r, k)
            assert float(np.max(np.abs(d["ranks"][k] - res.ranks))) <= 1e-13, (r, k)
