"""Fused K1+SpMV variants (occupancy x row parts) vs SpMV + plain K1 (R=1)."""
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
tsp = timed(lambda: eng.op.apply_ptr(eng.col_ptr(0), eng.col_ptr(1), None, None, -1, st), 10)
for p in (2, 4, 8, 13, 20, 26, 33, 40, 45, 51):
    row = []
    for occ, R in ((1, 1), (1, 2), (2, 1), (2, 2)):
        lib.lsb_set_tuning(1, occ)
        lib.lsb_set_tuning(2, R)
        tf = timed(lambda: lib.lsb_lagged_reduce_spmv7(S, C.byref(eng.op.c), 0, p, st), 10)
        row.append(f"o{3 if occ == 1 else 2}R{R} {1e3*tf:6.0f}")
    lib.lsb_set_tuning(1, 0)
    lib.lsb_set_tuning(2, 1)
    tk = timed(lambda: lib.lsb_lagged_reduce(S, 0, p, st), 10)
    lib.lsb_set_tuning(2, 0)
    print(f"p={p:3d}  " + "  ".join(row) + f"   | spmv+K1(R1) {1e3*(tk+tsp):6.0f} us")
