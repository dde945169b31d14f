"""Debug aid: run a small row-partitioned solve on in-process ranks with the
peer exchange and print each rank's exchange counters."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LSB_PEER_TIMEOUT_S", "5")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200.parallel import local_rhs, run_threads, slab_problem  # noqa: E402


def body(comm, N, kind, meth, m):
    op, ng = slab_problem((N, N, N), comm, kind=kind)
    b = local_rhs((N, N, N), comm, 42)
    cfg = P.GmresConfig(restart_m=m, max_restarts=20, rel_tol=1e-10, method=meth)
    try:
        x, h = P.gmres.solve_distributed(op, b, comm, ng, config=cfg)
        res = ("ok", h.iterations, h.outcome)
    except Exception as e:
        import traceback
        res = ("err", repr(e), traceback.format_exc()[-1500:])
    torch.cuda.synchronize()
    return res, comm.ctr.cpu().tolist(), comm.sig.cpu().tolist()


if __name__ == "__main__":
    ranks = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    kind = sys.argv[2] if len(sys.argv) > 2 else "convdiff27"
    N = int(sys.argv[3]) if len(sys.argv) > 3 else 16
    meth = sys.argv[4] if len(sys.argv) > 4 else "one_sync_mgs"
    m = int(sys.argv[5]) if len(sys.argv) > 5 else 100
    out = run_threads(ranks, body, N, kind, meth, m, peer=True)
    for r, o in enumerate(out):
        print(r, o)
