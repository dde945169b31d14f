"""Kernel timeline of graph-replayed GMRES cycles (CUPTI through
torch.profiler: real start/end times, no serialisation -- unlike an ncu
launch list): per-kernel totals, the idle gaps between consecutive kernels,
and the step's fraction of its HBM ceiling.

    python tools/timeline.py [--N 256] [--method two_sync_cgs2] [--cycles 2] [--m 50]
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--m", type=int, default=50)
    ap.add_argument("--method", default="two_sync_cgs2")
    ap.add_argument("--cycles", type=int, default=2)
    ap.add_argument("--out", default="")
    ap.add_argument("--seq", default="",
                    help="comma-separated kernel names: also record their per-launch "
                         "durations in launch order (first cycle)")
    a = ap.parse_args()
    A = P.gen_laplace3d(a.N)
    b = np.random.default_rng(42).standard_normal(A.n_rows)
    b /= np.linalg.norm(b)
    eng = Engine(A, a.m, a.method, 1e-14)
    eng.load(torch.as_tensor(b).cuda())
    eng.prologue()
    for _ in range(3):
        eng.cycle()                    # eager, then capture, then a replay
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.cycles):
            eng.cycle()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
           and e.name and not e.name.startswith("Memcpy") and not e.name.startswith("Memset")]
    evs.sort(key=lambda e: e.time_range.start)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    gaps = collections.defaultdict(float)
    span = (evs[-1].time_range.end - evs[0].time_range.start) if evs else 0
    busy = 0.0
    last_end = None
    want = set(x for x in a.seq.split(",") if x)
    seq = collections.defaultdict(list)
    for e in evs:
        nm = e.name.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        nm = nm.split("(")[0].replace("void ", "").replace("lsb::", "")
        nm = nm.split("<")[0]
        d = e.time_range.end - e.time_range.start
        tot[nm] += d
        cnt[nm] += 1
        if nm in want:
            seq[nm].append(round(d, 1))
        busy += d
        if last_end is not None and e.time_range.start > last_end:
            gaps[nm] += e.time_range.start - last_end   # idle before this kernel
        last_end = max(last_end or 0, e.time_range.end)
    out = {"method": a.method, "N": a.N, "m": a.m, "cycles": a.cycles,
           "span_us": span, "kernel_busy_us": busy,
           "idle_us": sum(gaps.values()),
           "kernels": {k: {"n": cnt[k], "total_us": round(tot[k], 1),
                           "avg_us": round(tot[k] / cnt[k], 2),
                           "idle_before_us": round(gaps[k], 1)} for k in tot}}
    if want:
        out["seq_us"] = dict(seq)
    print(json.dumps(out, indent=1))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
