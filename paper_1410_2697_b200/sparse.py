"""Sparse storage and the device sparse operator.

Mirrors the reference's ``SparseMatrix`` / ``AdjGraph`` / ``spmv`` /
``adjacency_graph`` (``/root/reference/pkg/src/mfhodlr/sparse.py:14-132,
277-291``). Storage is host CSC (validated, immutable, duplicates summed,
indices sorted) — the input format of the path; the adjacency graph is built
by the native library, and ``spmv`` runs on the GPU (CSR SpMV kernel).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import _lib


class SparseMatrix:
    """Real sparse matrix in compressed column-major storage (sparse.py:14-88)."""

    def __init__(self, matrix, symmetric=False):
        csc = sp.csc_matrix(matrix, dtype=np.float64)
        csc.sum_duplicates()
        csc.sort_indices()
        self._csc = csc
        self.symmetric = bool(symmetric)
        if self.symmetric:
            if csc.shape[0] != csc.shape[1]:
                raise ValueError("symmetric flag requires a square matrix")
            if (csc != csc.T).nnz != 0:
                raise ValueError("symmetric flag set but matrix is not symmetric")
        self._csr_cache = None
        self._dev = None

    @property
    def n_rows(self):
        return self._csc.shape[0]

    @property
    def n_cols(self):
        return self._csc.shape[1]

    @property
    def shape(self):
        return self._csc.shape

    @property
    def nnz(self):
        return self._csc.nnz

    @classmethod
    def from_triplets(cls, n_rows, n_cols, rows, cols, values, symmetric=False):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        values = np.asarray(values, dtype=np.float64)
        if rows.size and (rows.min() < 0 or rows.max() >= n_rows):
            raise ValueError("row index out of range")
        if cols.size and (cols.min() < 0 or cols.max() >= n_cols):
            raise ValueError("column index out of range")
        key = rows * n_cols + cols
        if np.unique(key).size != key.size:
            raise ValueError("duplicate (row, col) entry")
        return cls(sp.coo_matrix((values, (rows, cols)), shape=(n_rows, n_cols)), symmetric=symmetric)

    def to_csc(self):
        return self._csc.copy()

    def to_csr(self):
        return self._csc.tocsr()

    def csr_arrays(self):
        """(indptr, indices, data) of the CSR form, int64/float64, rows sorted."""
        if self._csr_cache is None:
            csr = self._csc.tocsr()
            csr.sort_indices()
            self._csr_cache = (_lib.i64(csr.indptr), _lib.i64(csr.indices), _lib.f64(csr.data))
        return self._csr_cache

    def toarray(self):
        return self._csc.toarray()

    def diagonal(self):
        return self._csc.diagonal()

    def device_operator(self):
        """The matrix uploaded as a device CSR operator (created once)."""
        if self._dev is None:
            self._dev = DeviceCsr(self)
        return self._dev

    def __repr__(self):
        return (f"SparseMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz},"
                f" symmetric={self.symmetric})")


class DeviceCsr:
    """mfh_csr: a matrix resident on the GPU for SpMV."""

    def __init__(self, A: SparseMatrix, ctx=None):
        import ctypes as C
        self.ctx = ctx or _lib.context()
        ip, ix, dv = A.csr_arrays()
        h = C.c_void_p()
        _lib.check(_lib.lib().mfh_csr_create(self.ctx.handle, A.n_rows, A.n_cols, _lib.ptr(ip),
                                             _lib.ptr(ix), _lib.ptr(dv), C.byref(h)))
        self.handle = h
        self.n_rows, self.n_cols = A.n_rows, A.n_cols
        _lib.register(self)

    def matvec(self, x):
        x = _lib.f64(x)
        y = np.empty(self.n_rows)
        _lib.check(_lib.lib().mfh_spmv(self.handle, _lib.ptr(x), _lib.ptr(y), 0))
        return y

    def _release(self):
        if self.handle and not _lib._finalized:
            _lib.lib().mfh_csr_free(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self._release()
        except Exception:
            pass


class DeviceDense:
    """Dense row-major operator on the GPU (LinearOperator.from_matrix(ndarray))."""

    def __init__(self, M, ctx=None):
        import ctypes as C
        self.ctx = ctx or _lib.context()
        M = np.ascontiguousarray(M, dtype=np.float64)
        if M.ndim != 2 or M.shape[0] != M.shape[1]:
            raise ValueError("dense operator must be square")
        h = C.c_void_p()
        _lib.check(_lib.lib().mfh_dense_create(self.ctx.handle, M.shape[0], _lib.ptr(M), C.byref(h)))
        self.handle = h
        self.n_rows = self.n_cols = M.shape[0]
        _lib.register(self)

    def matvec(self, x):
        x = _lib.f64(x)
        y = np.empty(self.n_rows)
        _lib.check(_lib.lib().mfh_spmv(self.handle, _lib.ptr(x), _lib.ptr(y), 0))
        return y

    def _release(self):
        if self.handle and not _lib._finalized:
            _lib.lib().mfh_csr_free(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self._release()
        except Exception:
            pass


class AdjGraph:
    """Undirected adjacency of a matrix pattern, self-loops removed (sparse.py:91-132)."""

    def __init__(self, n_vertices, indptr, indices):
        self.n_vertices = int(n_vertices)
        self.indptr = np.asarray(indptr, dtype=np.int64)
        self.indices = np.asarray(indices, dtype=np.int64)

    @classmethod
    def from_pattern(cls, pattern):
        """Symmetrize the nonzero-valued pattern and drop the diagonal (native)."""
        csr = sp.csr_matrix(pattern)
        csr.sort_indices()
        return _adjacency(csr.shape[0], _lib.i64(csr.indptr), _lib.i64(csr.indices),
                          _lib.f64(csr.data.astype(np.float64)))

    def neighbors(self, v):
        return self.indices[self.indptr[v]:self.indptr[v + 1]]

    def degree(self, v):
        return int(self.indptr[v + 1] - self.indptr[v])

    @property
    def n_edges(self):
        return int(len(self.indices) // 2)


def _adjacency(n, ip, ix, dv):
    import ctypes as C
    L = _lib.lib()
    nnz = C.c_int64()
    _lib.check(L.mfh_adjacency(n, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv), None, None, C.byref(nnz)))
    optr = np.empty(n + 1, dtype=np.int64)
    oidx = np.empty(max(1, nnz.value), dtype=np.int64)
    _lib.check(L.mfh_adjacency(n, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv), _lib.ptr(optr),
                               _lib.ptr(oidx), C.byref(nnz)))
    return AdjGraph(n, optr, oidx[:nnz.value])


def adjacency_graph(A: SparseMatrix):
    """Symmetrized pattern of a square matrix with the diagonal dropped (sparse.py:287-291)."""
    if A.n_rows != A.n_cols:
        raise ValueError("adjacency graph requires a square matrix")
    ip, ix, dv = A.csr_arrays()
    return _adjacency(A.n_rows, ip, ix, dv)


def spmv(A: SparseMatrix, x):
    """``A @ x`` on the GPU (sparse.py:277-284)."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[0] != A.n_cols:
        raise ValueError(
            f"dimension mismatch: matrix has {A.n_cols} columns, vector has {x.shape[0]}")
    return A.device_operator().matvec(x)
