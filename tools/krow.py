"""K2 (lagged update) vs persistent CTAs per SM (LSB_TUNE_ROW_CTAS_PER_SM)."""
import os, sys
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
eng.scal[_abi.S_BETA] = 1.0
eng.coef.fill_(1e-3)
st, S = D.stream(), eng.Sref
for p in (2, 10, 26, 51):
    row = []
    for c in (2, 3, 4, 5, 6, 8, 12, 16):
        lib.lsb_set_tuning(3, c)
        t = timed(lambda: lib.lsb_lagged_update(S, 0, p, 0, st), 10)
        row.append(f"{c}:{8*n*(p+3)/t/1e6:5.0f}")
    lib.lsb_set_tuning(3, 0)
    print(f"p={p:3d} " + " ".join(row))
