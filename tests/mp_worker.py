"""Worker for tests/test_multiproc_gpu.py: one rank of a 2-process fused
partition that shares cuda:0 with its peer.  Real CUDA IPC mappings between
the processes, peer stores and arrival counters from the pull kernel; the
host steps the loop (distributed.run_distributed(exchange="peer-host")) so no
kernel waits on the other process.  Writes its gathered ranks and per-lane
iterations to argv[1]."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    out, scale, alphas = sys.argv[1], int(sys.argv[2]), [float(a) for a in sys.argv[3].split(",")]
    exchange = sys.argv[4] if len(sys.argv) > 4 else "peer-host"
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    import paper_2108_02997_b200 as prl
    from paper_2108_02997_b200 import distributed
    g = prl.generate_rmat(scale, 16, 0.57, 0.19, 0.19, 2108, device=0)
    r = distributed.run_distributed(g, alphas, 1e-9, prl.NormKind.L1, 200, want_ranks=True,
                                    exchange=exchange)
    np.savez(out, ranks=r.ranks, iterations=r.iterations, sent=r.sent_bytes)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
