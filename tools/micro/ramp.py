import torch, json
flush = torch.ones(1 << 25, dtype=torch.float64, device="cuda")
sink = torch.empty((), dtype=torch.float64, device="cuda")
def cold(fn, reps=10):
    tot=0
    for _ in range(reps):
        torch.sum(flush, dim=0, out=sink)
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); tot+=e0.elapsed_time(e1)
    return round(1e3*tot/reps,2)
def warm(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return round(1e3*e0.elapsed_time(e1)/reps,2)
for mb in [1, 25, 50, 100, 200, 400, 800]:
    n = mb*2**20//8
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    s = torch.empty((), dtype=torch.float64, device="cuda")
    r = {"MB": mb, "sum_cold": cold(lambda: torch.sum(x, dim=0, out=s)),
         "copy_cold": cold(lambda: y.copy_(x)),
         "empty_kernel": cold(lambda: s.fill_(0))}
    r["sum_TBps"] = round(mb*2**20/r["sum_cold"]/1e6,2)
    r["copy_TBps"] = round(2*mb*2**20/r["copy_cold"]/1e6,2)
    print(json.dumps(r), flush=True)
