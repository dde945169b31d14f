"""Fused K1+SpMV (7-point, 256^3): pipelined stencil (LSB_TUNE_FUSED_PIPE 1:
forced wherever it compiles) vs the two-barrier kernel (2), next to plain K1,
at several p."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1809_05805_b200 as P
from paper_1809_05805_b200 import _abi, _dev as D
from paper_1809_05805_b200.engine import Engine
from kbench import timed

lib = _abi.load()
A = P.gen_laplace3d(256)
eng = Engine(A, 50, "one_sync_mgs", 1e-14, use_graph=False)
n = eng.n
eng.Vstore[:, :n].normal_(generator=torch.Generator(device="cuda").manual_seed(0))
eng.flags.copy_(torch.tensor([_abi.NO_STOP, 0, -1, 0, 0, 0, 0, 0], dtype=torch.int32))
st, S = D.stream(), eng.Sref
tot = {"pipe": 0.0, "old": 0.0, "k1": 0.0}
for p in [int(v) for v in os.environ.get("KPIPE_PS", "2,5,8,13,20,26,33,40,51").split(",")]:
    res = {}
    for name, knob in (("pipe", 1), ("old", 2)):
        lib.lsb_set_tuning(_abi.TUNE_FUSED_PIPE, knob)
        res[name] = timed(lambda: lib.lsb_lagged_reduce_spmv7(S, C.byref(eng.op.c), 0, p, st), 10)
    lib.lsb_set_tuning(_abi.TUNE_FUSED_PIPE, 0)
    tk = timed(lambda: lib.lsb_lagged_reduce(S, 0, p, st), 10)
    gb = 8 * n * (p + 1) / 1e6
    print(f"p={p:3d}  pipe {1e3*res['pipe']:6.0f} us ({gb/res['pipe']:5.0f} GB/s)  "
          f"two-barrier {1e3*res['old']:6.0f} us ({gb/res['old']:5.0f} GB/s)  K1 alone {1e3*tk:6.0f} us",
          flush=True)
