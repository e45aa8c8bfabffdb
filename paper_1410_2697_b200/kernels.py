"""Kernel plugin: ``full_pivot_lu`` on the GPU (reference _kernels/__init__.py:25,
_core.pyx:23-86).

``full_pivot_lu(block, eps, max_rank)`` keeps the reference signature and
returns ``(lu, row_perm, col_perm, rank, next_ratio)`` with ``lu`` in the
reference's physically permuted layout. ``full_pivot_lu_batched`` runs a whole
list of blocks in one launch (one CTA per block).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import PivotMonotonicityError

BACKEND = "cuda-sm100a"


def full_pivot_lu_batched(blocks, eps, max_ranks):
    """Batched complete-pivot LU; returns a list of reference-shaped tuples."""
    blocks = [np.ascontiguousarray(b, dtype=np.float64) for b in blocks]
    if not blocks:
        return []
    ms = np.array([b.shape[0] for b in blocks], dtype=np.int64)
    ns = np.array([b.shape[1] for b in blocks], dtype=np.int64)
    sizes = ms * ns
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    flat = np.concatenate([b.ravel() for b in blocks]) if sizes.sum() else np.zeros(1)
    flat = np.ascontiguousarray(flat, dtype=np.float64)
    caps = np.array([int(r) for r in max_ranks], dtype=np.int64)
    rp = np.empty(max(1, int(ms.sum())), dtype=np.int64)
    cp = np.empty(max(1, int(ns.sum())), dtype=np.int64)
    ranks = np.empty(len(blocks), dtype=np.int64)
    ratios = np.empty(len(blocks))
    status = np.empty(len(blocks), dtype=np.int64)
    err = np.empty(3 * len(blocks))
    _lib.check(_lib.lib().mfh_full_pivot_lu_batched(
        _lib.context().handle, len(blocks), _lib.ptr(offs), _lib.ptr(ms), _lib.ptr(ns),
        _lib.ptr(flat), int(sizes.sum()), float(eps), _lib.ptr(caps), _lib.ptr(rp), _lib.ptr(cp),
        _lib.ptr(ranks), _lib.ptr(ratios), _lib.ptr(status), _lib.ptr(err)))
    out = []
    ro = co = 0
    for q, b in enumerate(blocks):
        m, n = b.shape
        if status[q]:
            raise PivotMonotonicityError(
                "pivot %d magnitude %.3e exceeds twice the previous %.3e"
                % (int(err[3 * q]), err[3 * q + 1], err[3 * q + 2]))
        lu = flat[offs[q]:offs[q] + m * n].reshape(m, n).copy()
        out.append((lu, rp[ro:ro + m].copy(), cp[co:co + n].copy(), int(ranks[q]), float(ratios[q])))
        ro += m
        co += n
    return out


def full_pivot_lu(block, eps, max_rank):
    """Single-block form of the reference kernel signature."""
    b = np.array(block, dtype=np.float64, copy=True, order="C")
    m, n = b.shape
    if m == 0 or n == 0:
        return b, np.arange(m, dtype=np.int64), np.arange(n, dtype=np.int64), 0, 0.0
    return full_pivot_lu_batched([b], eps, [max_rank])[0]
