"""mf_factorize / mf_solve on the GPU — drop-in for the reference engine API.

Same entry points, parameters, statistics and error messages as
``/root/reference/pkg/src/mfhodlr/multifrontal.py:30-560``; the numeric
factorization and the two-pass solve run in ``libmfh.so`` (C-ABI
``mfh_factorize`` / ``mfh_apply``), batched by elimination-tree height.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .ordering import etree_handle
from .sparse import SparseMatrix

CONVENTIONAL = "conventional"
ACCELERATED = "accelerated"


@dataclass
class MfParams:
    """multifrontal.py:34-48"""

    n_c: int = 256
    eps: float = 1e-1
    d: int = 1
    n_leaf: int = 64
    max_rank: int | None = None


@dataclass
class FrontRecord:
    node_id: int
    front_size: int
    n_pivot: int
    path: str
    max_offdiag_rank: int
    stored_reals: int


_PATHS = {0: "empty", 1: "dense", 2: "structured"}


class FactorStats:
    """Per-node records plus the deterministic counters (multifrontal.py:61-112).

    ``records`` is materialized lazily from the raw int64 table (one row per
    node: node_id, front_size, n_pivot, path, max_offdiag_rank, stored_reals)."""

    def __init__(self, st, table):
        self._table = table
        self._records = None
        self.peak_stored_reals = int(st.peak_stored_reals)
        self.retained_reals = int(st.retained_reals)
        self.structured_fronts = int(st.structured_fronts)
        self.dense_fronts = int(st.dense_fronts)
        self.full_square_allocs = int(st.full_square_allocs)
        self.n_blocks = int(st.n_blocks)
        self.n_dense_fallback = int(st.n_dense_fallback)
        self.device_bytes = int(st.device_bytes_peak)

    @property
    def records(self):
        if self._records is None:
            self._records = [FrontRecord(int(r[0]), int(r[1]), int(r[2]), _PATHS[int(r[3])], int(r[4]), int(r[5]))
                             for r in self._table]
        return self._records

    def to_csv(self, path):
        with open(path, "w", encoding="ascii") as fh:
            fh.write("node_id,front_size,n_pivot,path,max_offdiag_rank,stored_reals\n")
            for r in self.records:
                fh.write(f"{r.node_id},{r.front_size},{r.n_pivot},{r.path},"
                         f"{r.max_offdiag_rank},{r.stored_reals}\n")


class NodeFactor:
    """DenseNodeFactor / StructuredNodeFactor (multifrontal.py:160-216) of one
    node: ids (pivots then frontal ids, permuted numbering), n_pivot, and the
    solve operators evaluated on the device factor."""

    def __init__(self, F, node_id, record):
        self._F = F
        self.node_id = node_id
        node = F.tree.nodes[node_id]
        self.ids = node.front_ids()
        self.n_pivot = node.n_pivot
        self.kind = record.path
        self._record = record

    def _op(self, op, v, n_out):
        v = np.ascontiguousarray(v, dtype=np.float64)
        y = np.empty(n_out)
        _lib.check(_lib.lib().mfh_node_op(self._F._h, self.node_id, op, _lib.ptr(v), _lib.ptr(y)))
        return y

    def pp_solve(self, v):
        return self._op(0, v, self.n_pivot)

    def apply_pf(self, v):
        return self._op(1, v, self.n_pivot)

    def apply_fp(self, v):
        return self._op(2, v, len(self.ids) - self.n_pivot)

    def stored_reals(self):
        return self._record.stored_reals

    def max_offdiag_rank(self):
        return self._record.max_offdiag_rank


class MfFactorization:
    """Device-resident factorization (multifrontal.py:227-242)."""

    def __init__(self, handle, mode, params, tree, ctx):
        self._h = handle
        self._ctx = ctx
        self.mode = mode
        self.params = params
        self.tree = tree
        self.permutation = tree.permutation
        self.n = tree.n
        L = _lib.lib()
        st = _lib.mfh_stats_t()
        _lib.check(L.mfh_factor_stats(handle, C.byref(st)))
        table = np.empty((max(1, st.n_records), 6), dtype=np.int64)
        _lib.check(L.mfh_factor_records(handle, _lib.ptr(table)))
        self.stats = FactorStats(st, table[:st.n_records])
        self._stored = int(st.stored_reals)
        self._node_factors = None
        _lib.register(self)

    def stored_reals(self):
        return self._stored

    @property
    def node_factors(self):
        """{node id: NodeFactor view, or None for empty fronts} (multifrontal.py:477-521).
        The operators run on the device factor (mfh_node_op)."""
        if self._node_factors is None:
            by_node = {r.node_id: r for r in self.stats.records}
            nf = {}
            for p in self.tree.post_order:
                r = by_node.get(p)
                nf[p] = None if r is None or r.path == "empty" else NodeFactor(self, p, r)
            self._node_factors = nf
        return self._node_factors

    def timing(self):
        t = _lib.mfh_timing_t()
        _lib.check(_lib.lib().mfh_factor_timing(self._h, C.byref(t)))
        return {k: getattr(t, k) for k, _ in t._fields_}

    def block_log(self):
        """Integer parity record of every compressed block, in the reference's
        visiting order: list of dicts (node, m, n, nI, nJ, rank, dense,
        row_perm, col_perm, ratio)."""
        L = _lib.lib()
        nb, npm = C.c_int64(), C.c_int64()
        _lib.check(L.mfh_factor_blocks(self._h, C.byref(nb), C.byref(npm), None, None, None))
        info = np.empty(7 * max(1, nb.value), dtype=np.int64)
        perms = np.empty(2 * max(1, npm.value), dtype=np.int64)
        ratios = np.empty(max(1, nb.value))
        _lib.check(L.mfh_factor_blocks(self._h, C.byref(nb), C.byref(npm), _lib.ptr(info),
                                       _lib.ptr(perms), _lib.ptr(ratios)))
        out, q = [], 0
        for b in range(nb.value):
            node, m, n, nI, nJ, rank, dense = (int(x) for x in info[7 * b:7 * b + 7])
            pr = perms[2 * q:2 * (q + rank)]
            out.append(dict(node=node, m=m, n=n, nI=nI, nJ=nJ, rank=rank, dense=bool(dense),
                            row_perm=pr[0::2].copy(), col_perm=pr[1::2].copy(), ratio=float(ratios[b])))
            q += rank
        return out

    def apply_bench(self, reps=20):
        ms, by = C.c_double(), C.c_double()
        _lib.check(_lib.lib().mfh_apply_bench(self._h, int(reps), C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def _release(self):
        if self._h and not _lib._finalized:
            _lib.lib().mfh_factor_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self._release()
        except Exception:
            pass


def mf_factorize(A, tree, mode=CONVENTIONAL, params=None):
    """Post-order multifrontal factorization on the GPU (multifrontal.py:459-530).

    ``mode='conventional'`` is the accelerated engine with the threshold at
    infinity: every front is dense.
    """
    if mode not in (CONVENTIONAL, ACCELERATED):
        raise ValueError(f"unknown mode '{mode}'")
    params = params or MfParams()
    if not isinstance(A, SparseMatrix):
        A = SparseMatrix(A)
    th = etree_handle(tree)  # ours, or the caller's own tree (e.g. the reference's) flattened as is
    ctx = _lib.context()
    ip, ix, dv = A.csr_arrays()
    p = _lib.mfh_params(int(min(params.n_c, 2**62)), float(params.eps), int(params.d),
                        int(params.n_leaf), -1 if params.max_rank is None else int(params.max_rank))
    h = C.c_void_p()
    _lib.check(_lib.lib().mfh_factorize(ctx.handle, th, A.n_rows, _lib.ptr(ip), _lib.ptr(ix),
                                        _lib.ptr(dv), 1 if mode == ACCELERATED else 0, C.byref(p),
                                        C.byref(h)))
    return MfFactorization(h, mode, params, tree, ctx)


def mf_solve(F, b):
    """Two-pass solve (multifrontal.py:533-560) as one CUDA-graph replay."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape[0] != F.n:
        raise ValueError(f"dimension mismatch: system is {F.n}, rhs is {b.shape[0]}")
    if b.ndim == 1:
        b = np.ascontiguousarray(b)
        x = np.empty(F.n)
        _lib.check(_lib.lib().mfh_apply(F._h, _lib.ptr(b), _lib.ptr(x), 1, 0))
        return x
    # several right-hand sides: columns
    bt = np.ascontiguousarray(b.T)
    xt = np.empty_like(bt)
    _lib.check(_lib.lib().mfh_apply(F._h, _lib.ptr(bt), _lib.ptr(xt), bt.shape[0], 0))
    return xt.T.copy()
