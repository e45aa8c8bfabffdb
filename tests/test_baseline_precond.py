"""Baseline preconditioners (krylov.py:164-214): ILUT factors
bit-identical to the reference's ilut_factor (_core.pyx:145-269; fixture
tests/golden/make_golden_ilut.py), the GPU applies bit-identical to the
reference's triangular-solve loops, diagonal scaling, GMRES with both."""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import REFERENCE_SRC
from paper_1410_2697_b200 import problems as PR

GENS = {
    "p7_8_k1": lambda: PR.gen_poisson7(8, 8, 8),
    "p7_10_k2": lambda: PR.gen_poisson7(10, 9, 8),
    "hex_6_k1": lambda: PR.gen_hex_q1(6, seed=2),
    "q1_20_k3": lambda: PR.gen_q1_2d(20),
    "p1_15_k1": lambda: PR.gen_p1_delaunay(15, seed=4),
}


def host_ilut(A, k, tol):
    """mfh_ilut_factor: the native host factorization (no GPU context)."""
    from paper_1410_2697_b200 import _lib
    ip, ix, dv = A.csr_arrays()
    n = A.n_rows
    lnz, unz = C.c_int64(), C.c_int64()
    L = _lib.lib()
    _lib.check(L.mfh_ilut_factor(n, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv), int(k), float(tol), C.byref(lnz),
                                 C.byref(unz), None, None, None, None, None, None))
    lp, up = np.empty(n + 1, np.int64), np.empty(n + 1, np.int64)
    li, lv = np.empty(max(1, lnz.value), np.int64), np.empty(max(1, lnz.value))
    ui, uv = np.empty(max(1, unz.value), np.int64), np.empty(max(1, unz.value))
    _lib.check(L.mfh_ilut_factor(n, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv), int(k), float(tol), C.byref(lnz),
                                 C.byref(unz), _lib.ptr(lp), _lib.ptr(li), _lib.ptr(lv), _lib.ptr(up),
                                 _lib.ptr(ui), _lib.ptr(uv)))
    return lp, li[:lnz.value], lv[:lnz.value], up, ui[:unz.value], uv[:unz.value]


@pytest.mark.parametrize("name", sorted(GENS))
def test_ilut_factors_bitwise(golden, name):
    g = golden("ilut.npz")
    A, _ = GENS[name]()
    k, tol, _ = g[f"{name}_meta"]
    got = host_ilut(A, int(k), float(tol))
    for part, arr in zip(("lp", "li", "lv", "up", "ui", "uv"), got):
        np.testing.assert_array_equal(arr, g[f"{name}_{part}"], err_msg=part)


def test_ilut_errors():
    from paper_1410_2697_b200 import _lib
    import scipy.sparse as sp
    from paper_1410_2697_b200.sparse import SparseMatrix
    A, _ = PR.gen_poisson7(3, 3, 3)
    with pytest.raises(ValueError, match="k must be at least 1"):
        host_ilut(A, 0, 1e-4)
    with pytest.raises(ValueError, match="drop_tol must be nonnegative"):
        host_ilut(A, 1, -1.0)
    Z = SparseMatrix(sp.csc_matrix(np.array([[0.0, 1.0], [1.0, 2.0]])))
    with pytest.raises(ValueError, match="ILUT zero pivot in row 0"):
        host_ilut(Z, 1, 0.0)


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not mounted (GPU box)")
def test_ilut_live_reference_random():
    """A fresh random nonsymmetric matrix (ties in magnitude included): the
    live reference's ilut_factor and ours agree bit for bit."""
    import importlib
    import sys
    import scipy.sparse as sp
    from paper_1410_2697_b200.sparse import SparseMatrix
    sys.path.insert(0, REFERENCE_SRC)
    try:
        mk = importlib.import_module("mfhodlr._kernels")
    finally:
        sys.path.remove(REFERENCE_SRC)
    rng = np.random.default_rng(7)
    n = 300
    M = sp.random(n, n, density=0.03, random_state=8, format="csr") + sp.eye(n) * 4
    M.data = np.round(M.data * 4) / 4  # magnitude ties
    A = SparseMatrix(M.tocsc())
    for k, tol in ((1, 1e-3), (2, 0.0), (4, 1e-1)):
        csr = A.to_csr()
        csr.sort_indices()
        ref = mk.ilut_factor(n, csr.indptr.astype(np.int64), csr.indices.astype(np.int64), csr.data,
                             int(k * A.nnz // n) + 1, tol)
        got = host_ilut(A, k, tol)
        for a, b in zip(got, ref):
            np.testing.assert_array_equal(a, b)
    del rng


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GENS))
def test_ilut_and_diag_apply_on_gpu(golden, name):
    import paper_1410_2697_b200 as P
    g = golden("ilut.npz")
    A, _ = GENS[name]()
    k, tol, stored = g[f"{name}_meta"]
    M = P.ilut(A, k=int(k), drop_tol=float(tol))
    assert M.stored_reals == int(stored)
    for part, arr in zip(("lp", "li", "lv"), M.l_parts):
        np.testing.assert_array_equal(arr, g[f"{name}_{part}"])
    b = g[f"{name}_b"]
    np.testing.assert_array_equal(M.apply_inverse(b), g[f"{name}_x"])  # level-scheduled GPU solves, bitwise
    D = P.diagonal_preconditioner(A)
    np.testing.assert_array_equal(D.apply_inverse(b), g[f"{name}_xdiag"])
    x, h = P.gmres(A, b, M=M, tol=1e-10, restart=30)
    ref = g[f"{name}_gmres_hist"]
    assert abs(h.iterations - len(ref)) <= 1 and h.converged
    np.testing.assert_allclose(h.residuals[:len(ref) - 1], ref[:len(h.residuals[:len(ref) - 1])], rtol=1e-6)
    xd, hd = P.gmres(A, b, M=D, tol=1e-10, restart=30)
    assert hd.converged and np.linalg.norm(A._csc @ xd - b) <= 1e-9 * np.linalg.norm(b)


@pytest.mark.gpu
def test_diag_zero_entry_message():
    import scipy.sparse as sp
    import paper_1410_2697_b200 as P
    Z = P.SparseMatrix(sp.csc_matrix(np.array([[1.0, 1.0], [1.0, 0.0]])))
    with pytest.raises(ValueError, match="zero diagonal entry at index 1"):
        P.diagonal_preconditioner(Z)
