"""Right-preconditioned restarted GMRES on the GPU (krylov.py:16-161).

``gmres`` keeps the reference's signature, history semantics and error
messages. The Arnoldi vectors, SpMV, modified Gram-Schmidt and the
preconditioner apply all run in ``libmfh.so`` (``mfh_gmres``); only the
(restart x restart) Hessenberg / Givens recurrence runs on the host. User
operators given as Python callables are reached through a host callback.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .sparse import DeviceCsr, DeviceDense, SparseMatrix

DEFAULT_TOL = 1e-6
DEFAULT_MAX_ITER = 4000
DEFAULT_RESTART = 100


class LinearOperator:
    """Dimension plus a deterministic linear apply (krylov.py:21-33)."""

    def __init__(self, dimension, apply):
        self.dimension = int(dimension)
        self.apply = apply
        self._device = None

    @classmethod
    def from_matrix(cls, A):
        if isinstance(A, SparseMatrix):
            dev = A.device_operator()
            op = cls(A.n_rows, dev.matvec)
            op._device = dev
            return op
        A = np.asarray(A, dtype=np.float64)
        dev = DeviceDense(A)
        op = cls(A.shape[0], dev.matvec)
        op._device = dev
        return op


class Preconditioner:
    """Approximate inverse with a provenance label (krylov.py:36-46)."""

    LABELS = ("diagonal", "ilut", "accelerated-mf", "none")

    def __init__(self, apply_inverse, label, stored_reals=0, factorization=None):
        if label not in self.LABELS:
            raise ValueError(f"unknown preconditioner label '{label}'")
        self.apply_inverse = apply_inverse
        self.label = label
        self.stored_reals = stored_reals
        self._factor = factorization


class DevicePrecond:
    """mfh_precond: a baseline preconditioner resident on the GPU."""

    def __init__(self, h, ctx):
        self._h = h
        self._ctx = ctx
        _lib.register(self)

    def info(self):
        st, ln, un, lv = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().mfh_precond_info(self._h, C.byref(st), C.byref(ln), C.byref(un), C.byref(lv)))
        return st.value, ln.value, un.value, lv.value

    def apply(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        y = np.empty_like(v)
        _lib.check(_lib.lib().mfh_precond_apply(self._h, _lib.ptr(v), _lib.ptr(y), 0))
        return y

    def _release(self):
        if self._h:
            _lib.lib().mfh_precond_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self._release()
        except Exception:
            pass


def diagonal_preconditioner(A):
    """Elementwise division by the matrix diagonal (krylov.py:164-170), on the
    GPU; ValueError on a zero diagonal entry."""
    if not isinstance(A, SparseMatrix):
        A = SparseMatrix(A)
    ip, ix, dv = A.csr_arrays()
    h = C.c_void_p()
    ctx = _lib.context()
    _lib.check(_lib.lib().mfh_precond_diag_create(ctx.handle, A.n_rows, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv),
                                                  C.byref(h)))
    dev = DevicePrecond(h, ctx)
    prec = Preconditioner(dev.apply, "diagonal", stored_reals=A.n_rows)
    prec._device = dev
    return prec


def ilut(A, k=1, drop_tol=1e-4):
    """Dual-threshold incomplete LU (krylov.py:173-204): factors bit-identical
    to the reference's ``ilut_factor`` (computed natively on the host: a
    row-sequential recurrence), the two triangular solves on the GPU by level
    sets (one graph replay per apply, bit-identical to the reference's loops).
    ``l_parts`` / ``u_parts`` hold the factors as the reference's do."""
    if k < 1:
        raise ValueError("k must be at least 1")
    if drop_tol < 0:
        raise ValueError("drop_tol must be nonnegative")
    if not isinstance(A, SparseMatrix):
        A = SparseMatrix(A)
    if A.n_rows != A.n_cols:
        raise ValueError("ILUT requires a square matrix")
    ip, ix, dv = A.csr_arrays()
    h = C.c_void_p()
    ctx = _lib.context()
    _lib.check(_lib.lib().mfh_precond_ilut_create(ctx.handle, A.n_rows, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv),
                                                  int(k), float(drop_tol), C.byref(h)))
    dev = DevicePrecond(h, ctx)
    stored, lnz, unz, _ = dev.info()
    n = A.n_rows
    lp, up = np.empty(n + 1, np.int64), np.empty(n + 1, np.int64)
    li, lv = np.empty(max(1, lnz), np.int64), np.empty(max(1, lnz))
    ui, uv = np.empty(max(1, unz), np.int64), np.empty(max(1, unz))
    _lib.check(_lib.lib().mfh_precond_ilut_factors(h, _lib.ptr(lp), _lib.ptr(li), _lib.ptr(lv), _lib.ptr(up),
                                                   _lib.ptr(ui), _lib.ptr(uv)))
    prec = Preconditioner(dev.apply, "ilut", stored_reals=stored)
    prec._device = dev
    prec.l_parts = (lp, li[:lnz], lv[:lnz])
    prec.u_parts = (up, ui[:unz], uv[:unz])
    return prec


def ilut_factors_as_csr(prec):
    """The ILUT factors as scipy matrices, unit diagonal added to L (krylov.py:207-214)."""
    import scipy.sparse as sp
    n = len(prec.l_parts[0]) - 1
    lp, li, lv = prec.l_parts
    up, ui, uv = prec.u_parts
    L = sp.csr_matrix((lv, li, lp), shape=(n, n)) + sp.eye(n, format="csr")
    U = sp.csr_matrix((uv, ui, up), shape=(n, n))
    return L, U


def identity_preconditioner():
    return Preconditioner(lambda v: v, "none")


def mf_preconditioner(F):
    """Device preconditioner from a GPU factorization (``mf_solve`` never leaves the device)."""
    from .multifrontal import mf_solve
    return Preconditioner(lambda v: mf_solve(F, v), "accelerated-mf",
                          stored_reals=F.stored_reals(), factorization=F)


@dataclass
class ConvergenceHistory:
    residuals: list = field(default_factory=list)
    converged: bool = False
    iterations: int = 0

    def to_csv(self, path):
        with open(path, "w", encoding="ascii") as fh:
            fh.write("iteration,relative_residual\n")
            for k, r in enumerate(self.residuals, start=1):
                fh.write(f"{k},{r!r}\n")


def _callback(fn, n, errors):
    def cb(_user, xp, yp):
        try:
            x = np.ctypeslib.as_array(xp, shape=(n,)).copy()
            y = np.asarray(fn(x), dtype=np.float64)
            if y.shape != (n,):
                raise ValueError("operator returned a vector of the wrong length")
            np.ctypeslib.as_array(yp, shape=(n,))[:] = y
        except Exception as e:  # surface after the native call returns
            errors.append(e)
            np.ctypeslib.as_array(yp, shape=(n,))[:] = np.nan
    return _lib.HOST_OP(cb)


def gmres(A, b, M=None, tol=DEFAULT_TOL, max_iter=DEFAULT_MAX_ITER, restart=DEFAULT_RESTART):
    """Restarted GMRES on ``A M^{-1}`` (krylov.py:68-161)."""
    if not (0.0 < tol < 1.0):
        raise ValueError("tol must lie in (0, 1)")
    if max_iter < 1 or restart < 1:
        raise ValueError("max_iter and restart must be positive")
    b = np.ascontiguousarray(b, dtype=np.float64)
    if isinstance(A, SparseMatrix):
        A = LinearOperator.from_matrix(A)
    n = A.dimension
    if b.shape[0] != n:
        raise ValueError("right-hand side does not match the operator dimension")
    ctx = _lib.context()
    errors = []
    ops = _lib.mfh_gmres_ops()
    keep = []
    if A._device is not None:
        ops.A = A._device.handle
    else:
        cb = _callback(A.apply, n, errors)
        keep.append(cb)
        ops.A_cb = cb
    if M is not None and getattr(M, "_factor", None) is not None:
        ops.M = M._factor._h
    elif M is not None and getattr(M, "_device", None) is not None:
        ops.P = M._device._h
    elif M is not None:
        cb = _callback(M.apply_inverse, n, errors)
        keep.append(cb)
        ops.M_cb = cb
    x = np.zeros(n)
    hist = np.empty(max(1, int(max_iter)))
    nh, its, conv = C.c_int64(), C.c_int64(), C.c_int()
    rc = _lib.lib().mfh_gmres(ctx.handle, C.byref(ops), n, _lib.ptr(b), _lib.ptr(x), float(tol),
                              int(max_iter), int(restart), _lib.ptr(hist), C.byref(nh), C.byref(its),
                              C.byref(conv))
    if errors:
        raise errors[0]
    _lib.check(rc)
    h = ConvergenceHistory([float(v) for v in hist[:nh.value]], bool(conv.value), int(its.value))
    return x, h


def gmres_batched(A, B, M, tol=DEFAULT_TOL, max_iter=DEFAULT_MAX_ITER, restart=DEFAULT_RESTART):
    """``gmres`` for the columns of ``B`` (n x k) with one device factorization:
    groups of up to eight right-hand sides run in lockstep and share each
    preconditioner apply (the factor is read once per Arnoldi step, not once per
    column, on the FP64 tensor cores). Every column equals
    ``gmres(A, B[:, j], M)`` to rounding (iteration counts within one) and does
    not depend on the other columns. ``A`` must be a SparseMatrix (or a LinearOperator
    from one) and ``M`` a ``mf_preconditioner``."""
    if not (0.0 < tol < 1.0):
        raise ValueError("tol must lie in (0, 1)")
    if max_iter < 1 or restart < 1:
        raise ValueError("max_iter and restart must be positive")
    if isinstance(A, SparseMatrix):
        A = LinearOperator.from_matrix(A)
    if A._device is None or M is None or getattr(M, "_factor", None) is None:
        raise ValueError("gmres_batched needs a device operator and an mf_preconditioner")
    B = np.asarray(B, dtype=np.float64)
    if B.ndim != 2 or B.shape[0] != A.dimension:
        raise ValueError("right-hand sides must be an (n, k) array matching the operator dimension")
    n, k = B.shape
    Bt = np.ascontiguousarray(B.T)
    Xt = np.zeros_like(Bt)
    ops = _lib.mfh_gmres_ops()
    ops.A = A._device.handle
    ops.M = M._factor._h
    cap = max(1, int(max_iter))
    hist = np.empty((max(1, k), cap))
    nh = np.zeros(max(1, k), dtype=np.int64)
    its = np.zeros(max(1, k), dtype=np.int64)
    conv = np.zeros(max(1, k), dtype=np.int32)
    _lib.check(_lib.lib().mfh_gmres_batched(_lib.context().handle, C.byref(ops), n, k, _lib.ptr(Bt), _lib.ptr(Xt),
                                            float(tol), int(max_iter), int(restart), _lib.ptr(hist), cap,
                                            _lib.ptr(nh), _lib.ptr(its), _lib.ptr(conv)))
    hs = [ConvergenceHistory([float(v) for v in hist[j, :nh[j]]], bool(conv[j]), int(its[j])) for j in range(k)]
    return Xt.T.copy(), hs
