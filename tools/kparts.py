"""Sweep K1 / fused row-part choices (LSB_TUNE_FORCE_PARTS) at C2 scale."""
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
for p in (6, 13, 20, 26, 33, 40, 45, 51):
    row = []
    for R in (1, 2, 4, 8):
        lib.lsb_set_tuning(2, R)
        tf = timed(lambda: lib.lsb_lagged_reduce_spmv7(S, C.byref(eng.op.c), 0, p, st), 10)
        tk = timed(lambda: lib.lsb_lagged_reduce(S, 0, p, st), 10)
        row.append(f"R={R}: {8*n*(p+1)/tf/1e6:6.0f}/{8*n*(p+1)/tk/1e6:6.0f}")
    lib.lsb_set_tuning(2, 0)
    print(f"p={p:3d}  " + "  ".join(row) + "   (fused/plain GB/s)")
