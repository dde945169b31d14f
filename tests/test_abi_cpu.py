"""CPU checks of the C-ABI boundary: liblsb200.so builds for sm_100a, loads,
and exports every entry point declared in include/lsb200.h; the ctypes
struct mirrors match the C layout; the product fails loudly without a GPU."""

import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lsb200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1809_05805_b200 import _abi, build
    build.build()
    return _abi.load()


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lsb_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    from paper_1809_05805_b200 import _abi
    assert set(names) == set(_abi.EXPORTS)


def test_nm_shows_extern_c_symbols(lib):
    from paper_1809_05805_b200 import _abi
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    for n in _declared():
        assert re.search(rf"\bT {n}$", out, re.M), n


def test_sass_is_sm100a(lib):
    from paper_1809_05805_b200 import _abi
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_c():
    """Compile a tiny C program printing sizeof/offsetof of the ABI structs
    and compare with the ctypes mirrors."""
    from paper_1809_05805_b200 import _abi
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "lsb200.h"
int main(void){
 printf("%zu %zu %zu %zu %zu\n", sizeof(lsb_flags), sizeof(lsb_workspace), sizeof(lsb_csr),
        sizeof(lsb_stencil), sizeof(lsb_arnoldi));
 printf("%zu %zu %zu %zu\n", offsetof(lsb_arnoldi, G), offsetof(lsb_arnoldi, Gloc),
        offsetof(lsb_arnoldi, ws), offsetof(lsb_stencil, col_scale));
 printf("%zu %zu %zu %zu %zu %zu\n", sizeof(lsb_peer), offsetof(lsb_peer, timeout_ns),
        offsetof(lsb_peer, sig), offsetof(lsb_peer, epoch), offsetof(lsb_peer, counter),
        offsetof(lsb_flags, comm_error));
 return 0;}
"""
    d = "/tmp/lsb_abi_check"
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "a.c"), "w") as fh:
        fh.write(prog)
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o",
                           os.path.join(d, "a.out"), os.path.join(d, "a.c")])
    out = subprocess.run([os.path.join(d, "a.out")], capture_output=True, text=True).stdout.split()
    sizes = [int(v) for v in out[:5]]
    offs = [int(v) for v in out[5:9]]
    peer = [int(v) for v in out[9:]]
    assert peer == [C.sizeof(_abi.Peer), _abi.Peer.timeout_ns.offset, _abi.Peer.sig.offset,
                    _abi.Peer.epoch.offset, _abi.Peer.counter.offset, _abi.Flags.comm_error.offset]
    assert sizes == [C.sizeof(_abi.Flags), C.sizeof(_abi.Workspace), C.sizeof(_abi.Csr),
                     C.sizeof(_abi.Stencil), C.sizeof(_abi.Arnoldi)]
    assert offs == [_abi.Arnoldi.G.offset, _abi.Arnoldi.Gloc.offset, _abi.Arnoldi.ws.offset,
                    _abi.Stencil.col_scale.offset]


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_1809_05805_b200 as P
    from paper_1809_05805_b200._abi import LsbUnavailable
    A = P.gen_laplace2d(4)
    with pytest.raises(LsbUnavailable):
        P.spmv(A, np.ones(16))
    with pytest.raises(LsbUnavailable):
        P.solve(A, np.ones(16))


def test_host_logic_without_gpu():
    """Ledger, config validation, CSR construction/validation and the
    stencil's CSR view are host logic and work on CPU."""
    import numpy as np
    import paper_1809_05805_b200 as P
    from oracle import lowsync_oracle as orc
    led = P.ReductionLedger()
    led.iteration = 3
    led.record("norm", 1)
    led.iteration = 4
    led.record("dot", 1)
    led.record("dot", 1)
    assert led.counts_per_iteration() == {3: 1, 4: 2}
    with pytest.raises(ValueError):
        led.record("allreduce", 1)
    assert P.canonical_method("one-sync") == "one_sync_mgs"
    with pytest.raises(ValueError):
        P.GmresConfig(restart_m=0)
    with pytest.raises(ValueError):
        P.CsrMatrix(1, 3, [0, 2], [2, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        P.CsrMatrix(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])
    A = P.CsrMatrix.from_coo(2, 2, [1, 0, 1, 1], [0, 0, 0, 1], [1.0, 2.0, 3.0, 4.0])
    assert A.nnz == 3 and A.to_dense()[1, 0] == 4.0
    for gen, ref in ((P.gen_laplace2d(9), orc.laplace2d(9)),
                     (P.gen_laplace3d(5), orc.laplace3d(5)),
                     (P.gen_convdiff27(4), orc.convdiff27(4))):
        assert np.array_equal(gen.row_ptr, ref.row_ptr)
        assert np.array_equal(gen.col_idx, ref.col_idx)
        assert np.array_equal(gen.values, ref.values)
        assert gen.nnz == ref.nnz
        assert abs(gen.frobenius_norm() - float(np.sqrt(np.dot(ref.values, ref.values)))) < 1e-9
