"""Host-side problem ingestion: Matrix Market loader (reference
harness.py:41-102, its tests test_harness.py:84-145) and generators."""

import numpy as np
import pytest

import paper_1809_05805_b200 as P
from oracle import lowsync_oracle as orc

IDENTITY = """%%MatrixMarket matrix coordinate real general
3 3 3
1 1 1.0
2 2 1.0
3 3 1.0
"""

SYMMETRIC = """%%MatrixMarket matrix coordinate real symmetric
% lower triangle only
3 3 4
1 1 2.0
2 1 -1.0
2 2 2.0
3 3 2.0
"""


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_identity(tmp_path):
    A = P.load_matrix_market(_write(tmp_path, "eye.mtx", IDENTITY))
    assert list(A.row_ptr) == [0, 1, 2, 3]
    assert np.array_equal(A.to_dense(), np.eye(3))


def test_symmetric_expansion(tmp_path):
    A = P.load_matrix_market(_write(tmp_path, "sym.mtx", SYMMETRIC))
    assert A.nnz == 5
    M = A.to_dense()
    assert M[0, 1] == M[1, 0] == -1.0


@pytest.mark.parametrize("text,match", [
    ("%%NotMatrixMarket stuff\n1 1 1\n1 1 1.0\n", "malformed"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0 0.0\n", "complex"),
    ("%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n", "pattern"),
    ("%%MatrixMarket matrix array real general\n2 2\n1.0\n0.0\n0.0\n1.0\n", "coordinate"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n", "declared"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "out of range"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", "bad entry"),
])
def test_rejections(tmp_path, text, match):
    with pytest.raises(P.MatrixMarketError, match=match):
        P.load_matrix_market(_write(tmp_path, "bad.mtx", text))


def test_duplicates_summed(tmp_path):
    A = P.load_matrix_market(_write(
        tmp_path, "dup.mtx",
        "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.5\n1 1 2.5\n2 2 1.0\n"))
    assert A.to_dense()[0, 0] == 4.0


def test_round_trip_matches_oracle_csr(tmp_path):
    """A 27-point operator written as a symmetric-free general file and read
    back reproduces the oracle's CSR bit for bit."""
    O = orc.convdiff27(5)
    rows = np.repeat(np.arange(O.n_rows), np.diff(O.row_ptr))
    lines = [f"{r + 1} {c + 1} {float(v)!r}" for r, c, v in zip(rows, O.col_idx, O.values)]
    text = (f"%%MatrixMarket matrix coordinate real general\n% c5\n{O.n_rows} {O.n_cols} "
            f"{O.nnz}\n" + "\n".join(lines) + "\n")
    A = P.load_matrix_market(_write(tmp_path, "c27.mtx", text))
    assert np.array_equal(A.row_ptr, O.row_ptr)
    assert np.array_equal(A.col_idx, O.col_idx)
    assert np.array_equal(A.values, O.values)


def test_generators():
    A = P.gen_simoncini(3)
    assert np.array_equal(A.diagonal_values(), [1e-8, 2.0, 3.0])
    assert P.gen_simoncini().nnz == 100
    L = P.gen_laplace2d(3)
    assert L.to_dense()[4, 4] == 4.0 and L.n_rows == 9
    b = P.gen_rhs("random", L, 42)
    assert abs(np.linalg.norm(b) - 1.0) < 1e-15
    assert np.array_equal(b, P.gen_rhs("random", L, 42))
    with pytest.raises(ValueError):
        P.gen_rhs("random", L, None)
