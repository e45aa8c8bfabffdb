"""Matrix Market interchange and row scaling (sparse.py:142-274): round trips,
the reference's validation messages, and agreement with the live reference
when it is mounted."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import REFERENCE_SRC
from paper_1410_2697_b200 import problems as PR
from paper_1410_2697_b200.mmio import load_matrix_market, row_scale, write_matrix_market
from paper_1410_2697_b200.sparse import SparseMatrix

BAD = {
    "empty": ("", "{p}:1: empty file"),
    "header": ("%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1.0\n", "{p}:1: missing '%%MatrixMarket' header"),
    "array": ("%%MatrixMarket matrix array real general\n1 1\n1.0\n",
              "{p}:1: unsupported header '%%MatrixMarket matrix array real general' (need coordinate matrix)"),
    "complex": ("%%MatrixMarket matrix coordinate complex general\n", "{p}:1: unsupported field 'complex' (only real is accepted)"),
    "herm": ("%%MatrixMarket matrix coordinate real hermitian\n", "{p}:1: unsupported symmetry 'hermitian'"),
    "nosize": ("%%MatrixMarket matrix coordinate real general\n% only a comment\n", "{p}:2: missing size line"),
    "badsize": ("%%MatrixMarket matrix coordinate real general\n%c\n2 2\n", "{p}:3: malformed size line '2 2'"),
    "symrect": ("%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1\n", "{p}:2: symmetric matrix must be square"),
    "malformed": ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 x 3\n", "{p}:4: malformed entry line '2 x 3'"),
    "range": ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n3 1 1\n", "{p}:4: entry (3, 1) out of range for 2x2"),
    "dup": ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 1\n\n1 1 5\n", "{p}:6: duplicate entry (1, 1)"),
    "upper": ("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1.0\n1 2 1\n", "{p}:4: symmetric file stores an entry above the diagonal"),
    "more": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1\n", "{p}: entry count mismatch: header declares 1, file has more"),
    "fewer": ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 1\n", "{p}: entry count mismatch: header declares 3, file has 2"),
    "comment_in_body": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n% late\n1 1 1.0\n", "{p}:3: malformed entry line '% late'"),
}


def _reference():
    import importlib
    import sys
    sys.path.insert(0, REFERENCE_SRC)
    try:
        return importlib.import_module("mfhodlr.sparse")
    finally:
        sys.path.remove(REFERENCE_SRC)


@pytest.mark.parametrize("name", sorted(BAD))
def test_validation_messages(tmp_path, name):
    text, msg = BAD[name]
    p = tmp_path / f"{name}.mtx"
    p.write_text(text)
    with pytest.raises(ValueError) as e:
        load_matrix_market(str(p))
    assert str(e.value) == msg.format(p=p)
    if os.path.isdir(REFERENCE_SRC):  # the reference's own text, live
        with pytest.raises(ValueError) as r:
            _reference().load_matrix_market(str(p))
        assert str(r.value) == str(e.value)


@pytest.mark.parametrize("sym", [True, False])
def test_round_trip(tmp_path, sym):
    if sym:
        A, _ = PR.gen_poisson7(5, 4, 3)
    else:
        rng = np.random.default_rng(2)
        M = sp.random(30, 20, density=0.2, random_state=3, format="csc")
        M.data = rng.standard_normal(M.nnz) * 10.0 ** rng.integers(-20, 20, M.nnz)
        A = SparseMatrix(M)
    p = tmp_path / "a.mtx"
    write_matrix_market(A, str(p))
    B = load_matrix_market(str(p))
    assert B.symmetric == A.symmetric and B.shape == A.shape
    assert (abs(A._csc - B._csc)).nnz == 0  # bit-exact values (shortest round-trip repr)
    if os.path.isdir(REFERENCE_SRC):
        R = _reference().load_matrix_market(str(p))
        assert R.symmetric == B.symmetric and (abs(R.to_csc() - B._csc)).nnz == 0
        q = tmp_path / "r.mtx"
        _reference().write_matrix_market(R, str(q))
        assert q.read_text() == p.read_text()


def test_row_scale():
    A, b = PR.gen_poisson7(4, 3, 3)
    As, bs, rec = row_scale(A, b)
    assert not As.symmetric
    np.testing.assert_array_equal(rec.row_scales, np.abs(A.to_csr()).max(axis=1).toarray().ravel())
    np.testing.assert_array_equal(np.abs(As.to_csr()).max(axis=1).toarray().ravel(), np.ones(A.n_rows))
    np.testing.assert_array_equal(bs, b / rec.row_scales)
    Z = SparseMatrix(sp.csc_matrix(np.array([[1.0, 0.0], [0.0, 0.0]])))
    with pytest.raises(ValueError, match="row 1 has no nonzero entries"):
        row_scale(Z, np.ones(2))
    with pytest.raises(ValueError, match="right-hand side length"):
        row_scale(A, np.ones(3))
    if os.path.isdir(REFERENCE_SRC):
        R = _reference()
        Ar, br, rr = R.row_scale(R.SparseMatrix(A._csc.copy(), symmetric=True), b)
        np.testing.assert_array_equal(br, bs)
        np.testing.assert_array_equal(rr.row_scales, rec.row_scales)
        assert (abs(Ar.to_csc() - As._csc)).nnz == 0
