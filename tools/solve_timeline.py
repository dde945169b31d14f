"""CUPTI timeline of one whole solve() (default 3D 7-point 32^3 one-sync
GMRES(50), tol 1e-6): every kernel with its start offset and duration, and
the idle gaps (host work between launches / report syncs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32
A = P.gen_laplace3d(N)
b = P.gen_rhs("random", A, 42)
cfg = P.GmresConfig(restart_m=50, max_restarts=50, rel_tol=1e-6)
for _ in range(3):
    x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
    h.release()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
last = t0
idle = 0.0
for e in evs:
    gap = e.time_range.start - last
    if gap > 0:
        idle += gap
    nm = e.name.split("(")[0].replace("void ", "").replace("lsb::", "")[:40]
    print(f"{e.time_range.start - t0:9.1f} +{gap:7.1f} {e.time_range.end - e.time_range.start:8.1f} {nm}")
    last = max(last, e.time_range.end)
print(f"span {last - t0:.1f} us, idle {idle:.1f} us, kernels {len(evs)}")
