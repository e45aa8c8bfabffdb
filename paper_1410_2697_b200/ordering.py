"""Nested dissection and elimination tree — native host symbolic analysis.

Same objects and integer results as the reference
(``/root/reference/pkg/src/mfhodlr/ordering.py:19-312``): ``SepNode`` /
``SeparatorTree`` / ``EtNode`` / ``EliminationTree``, built by the C++ code in
``csrc/symbolic.cpp`` (iterative, bit-identical permutation and index sets).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib

DEFAULT_LEAF_SIZE = 64


@dataclass
class SepNode:
    vertices: np.ndarray
    children: tuple | None = None
    parent: int | None = None

    @property
    def is_leaf(self):
        return self.children is None


class SeparatorTree:
    def __init__(self, nodes, root, permutation, handle=None):
        self.nodes = nodes
        self.root = root
        self.permutation = permutation
        self.n = len(permutation)
        self._h = handle

    def post_order(self):
        order = []
        if self.root is None:
            return order
        stack = [(self.root, False)]
        while stack:
            v, done = stack.pop()
            if done:
                order.append(v)
                continue
            stack.append((v, True))
            ch = self.nodes[v].children
            if ch is not None:
                stack.append((ch[1], False))
                stack.append((ch[0], False))
        return order

    def __del__(self):
        try:
            if self._h:
                _lib.lib().mfh_nd_free(self._h)
                self._h = None
        except Exception:
            pass


def nested_dissection(g, leaf_size=DEFAULT_LEAF_SIZE):
    """BFS level-set nested dissection (ordering.py:157-208), native."""
    if leaf_size < 1:
        raise ValueError("leaf_size must be at least 1")
    L = _lib.lib()
    ip, ix = _lib.i64(g.indptr), _lib.i64(g.indices)
    h = C.c_void_p()
    _lib.check(L.mfh_nd_create(g.n_vertices, _lib.ptr(ip), _lib.ptr(ix), int(leaf_size), C.byref(h)))
    nn, nv, root = C.c_int64(), C.c_int64(), C.c_int64()
    _lib.check(L.mfh_nd_sizes(h, C.byref(nn), C.byref(nv), C.byref(root)))
    nn, nv = nn.value, nv.value
    perm = np.empty(g.n_vertices, dtype=np.int64)
    vptr = np.empty(nn + 1, dtype=np.int64)
    verts = np.empty(max(1, nv), dtype=np.int64)
    left = np.empty(max(1, nn), dtype=np.int64)
    right = np.empty(max(1, nn), dtype=np.int64)
    parent = np.empty(max(1, nn), dtype=np.int64)
    _lib.check(L.mfh_nd_fetch(h, _lib.ptr(perm), _lib.ptr(vptr), _lib.ptr(verts), _lib.ptr(left),
                              _lib.ptr(right), _lib.ptr(parent)))
    nodes = []
    for v in range(nn):
        ch = None if left[v] < 0 else (int(left[v]), int(right[v]))
        par = None if parent[v] < 0 else int(parent[v])
        nodes.append(SepNode(verts[vptr[v]:vptr[v + 1]].copy(), ch, par))
    return SeparatorTree(nodes, None if nn == 0 else int(root.value), perm, h)


@dataclass
class EtNode:
    id: int
    pivot_ids: np.ndarray
    coupled_ids: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    frontal_ids: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    children: list = field(default_factory=list)
    parent: int | None = None

    @property
    def n_pivot(self):
        return len(self.pivot_ids)

    @property
    def front_size(self):
        return len(self.pivot_ids) + len(self.frontal_ids)

    def front_ids(self):
        return np.concatenate([self.pivot_ids, self.frontal_ids])


class EliminationTree:
    def __init__(self, nodes, post_order, permutation, root, handle=None):
        self.nodes = nodes
        self.post_order = post_order
        self.permutation = permutation
        self.root = root
        self.n = len(permutation)
        self._h = handle

    def outline(self):
        lines = []
        if self.root is None:
            return ""
        stack = [(self.root, 0)]
        while stack:
            v, d = stack.pop()
            nd = self.nodes[v]
            lines.append("  " * d + f"node {v}: |pivots|={nd.n_pivot} |frontal|={len(nd.frontal_ids)}")
            for c in reversed(nd.children):
                stack.append((c, d + 1))
        return "\n".join(lines)

    def __del__(self):
        try:
            if self._h:
                _lib.lib().mfh_etree_free(self._h)
                self._h = None
        except Exception:
            pass


def build_elimination_tree(tree, A):
    """Pivot / frontal index sets per node (ordering.py:264-312), native."""
    if tree.n != A.n_rows or A.n_rows != A.n_cols:
        raise ValueError("separator tree size does not match the matrix")
    if tree._h is None:
        raise ValueError("separator tree must come from nested_dissection")
    L = _lib.lib()
    ip, ix, dv = A.csr_arrays()
    h = C.c_void_p()
    _lib.check(L.mfh_etree_create(A.n_rows, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv), tree._h,
                                  C.byref(h)))
    nn, npv, nfr, root = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _lib.check(L.mfh_etree_sizes(h, C.byref(nn), C.byref(npv), C.byref(nfr), C.byref(root)))
    nn = nn.value
    post = np.empty(max(1, nn), dtype=np.int64)
    pptr = np.empty(nn + 1, dtype=np.int64)
    piv = np.empty(max(1, npv.value), dtype=np.int64)
    fptr = np.empty(nn + 1, dtype=np.int64)
    fr = np.empty(max(1, nfr.value), dtype=np.int64)
    par = np.empty(max(1, nn), dtype=np.int64)
    _lib.check(L.mfh_etree_fetch(h, _lib.ptr(post), _lib.ptr(pptr), _lib.ptr(piv), _lib.ptr(fptr),
                                 _lib.ptr(fr), _lib.ptr(par)))
    perm = tree.permutation
    nodes = [None] * nn
    for v in range(nn):
        sn = tree.nodes[v]
        et = EtNode(id=v, pivot_ids=piv[pptr[v]:pptr[v + 1]].copy())
        et.frontal_ids = fr[fptr[v]:fptr[v + 1]].copy()
        if len(et.pivot_ids):
            et.coupled_ids = np.zeros(0, dtype=np.int64)  # not materialized (frontal covers it)
        et.parent = None if par[v] < 0 else int(par[v])
        if sn.children is not None:
            et.children = list(sn.children)
        nodes[v] = et
    post_order = [int(p) for p in post[:nn]]
    return EliminationTree(nodes, post_order, perm, tree.root, h)


class _ForeignTree:
    """Owns the native copy of a caller-built elimination tree."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h:
                _lib.lib().mfh_etree_free(self.h)
                self.h = None
        except Exception:
            pass


def etree_handle(tree):
    """The native elimination tree for ``tree``: its own handle when it came
    from ``build_elimination_tree``; otherwise (e.g. the reference's
    ``EliminationTree``, ordering.py:238-261) the caller's tree is flattened
    and handed over as is through ``mfh_etree_from_arrays`` -- nothing is
    recomputed, so any leaf size or ordering the caller used is honoured."""
    h = getattr(tree, "_h", None)
    if h:
        return h
    cached = getattr(tree, "_mfh_foreign", None)
    if cached is not None:
        return cached.h
    nodes = tree.nodes
    nn = len(nodes)
    perm = np.ascontiguousarray(np.asarray(tree.permutation, dtype=np.int64))
    parent = np.full(max(1, nn), -1, dtype=np.int64)
    cptr = np.zeros(nn + 1, dtype=np.int64)
    kids, pivs, frs = [], [], []
    pptr = np.zeros(nn + 1, dtype=np.int64)
    fptr = np.zeros(nn + 1, dtype=np.int64)
    for v in range(nn):
        nd = nodes[v]
        ch = [] if nd is None else list(nd.children or [])
        pv = np.zeros(0, np.int64) if nd is None else np.asarray(nd.pivot_ids, dtype=np.int64)
        fr = np.zeros(0, np.int64) if nd is None else np.asarray(nd.frontal_ids, dtype=np.int64)
        if nd is not None and nd.parent is not None:
            parent[v] = int(nd.parent)
        kids += [int(c) for c in ch]
        pivs.append(pv)
        frs.append(fr)
        cptr[v + 1] = cptr[v] + len(ch)
        pptr[v + 1] = pptr[v] + len(pv)
        fptr[v + 1] = fptr[v] + len(fr)
    child = np.array(kids if kids else [0], dtype=np.int64)
    piv = np.concatenate(pivs) if pptr[-1] else np.zeros(1, np.int64)
    fr = np.concatenate(frs) if fptr[-1] else np.zeros(1, np.int64)
    post = np.array(list(tree.post_order) or [0], dtype=np.int64)
    root = -1 if tree.root is None else int(tree.root)
    h = C.c_void_p()
    _lib.check(_lib.lib().mfh_etree_from_arrays(len(perm), _lib.ptr(perm), nn, root, _lib.ptr(parent),
                                                _lib.ptr(cptr), _lib.ptr(child), len(tree.post_order),
                                                _lib.ptr(post), _lib.ptr(pptr), _lib.ptr(piv), _lib.ptr(fptr),
                                                _lib.ptr(fr), C.byref(h)))
    owner = _ForeignTree(h)
    try:
        tree._mfh_foreign = owner
    except AttributeError:
        pass
    return owner.h
