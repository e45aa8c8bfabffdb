"""The drop-in boundary takes the CALLER's elimination tree (SURVEY 8(b)
mfh_plan_create): mfh_etree_from_arrays receives the
reference's own EliminationTree (ordering.py:238-261) flattened, validates it,
and the factorization uses exactly that tree -- any ND leaf size the caller
chose is honoured. Fixture: tests/golden/make_golden_etree.py (the reference's
tree at ND leaf 40, its mf_solve on it)."""
import ctypes as C
import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import REFERENCE_SRC


def foreign_tree(g):
    """A reference-shaped EliminationTree (plain attributes, no native handle)."""
    nn = len(g["parent"])
    nodes = []
    for v in range(nn):
        nodes.append(SimpleNamespace(
            id=v, pivot_ids=g["piv"][g["pptr"][v]:g["pptr"][v + 1]],
            frontal_ids=g["fr"][g["fptr"][v]:g["fptr"][v + 1]],
            children=[int(c) for c in g["child"][g["cptr"][v]:g["cptr"][v + 1]]],
            parent=None if g["parent"][v] < 0 else int(g["parent"][v])))
    return SimpleNamespace(nodes=nodes, post_order=[int(p) for p in g["post"]], permutation=g["perm"],
                           root=int(g["root"]), n=len(g["perm"]))


def fetch(h):
    from paper_1410_2697_b200 import _lib
    L = _lib.lib()
    nn, npv, nfr, root = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _lib.check(L.mfh_etree_sizes(h, C.byref(nn), C.byref(npv), C.byref(nfr), C.byref(root)))
    nn = nn.value
    post, pptr, fptr, par = (np.empty(max(1, nn), np.int64), np.empty(nn + 1, np.int64), np.empty(nn + 1, np.int64),
                             np.empty(max(1, nn), np.int64))
    piv, fr = np.empty(max(1, npv.value), np.int64), np.empty(max(1, nfr.value), np.int64)
    _lib.check(L.mfh_etree_fetch(h, _lib.ptr(post), _lib.ptr(pptr), _lib.ptr(piv), _lib.ptr(fptr), _lib.ptr(fr),
                                 _lib.ptr(par)))
    return dict(post=post[:nn], pptr=pptr, piv=piv[:npv.value], fptr=fptr, fr=fr[:nfr.value], parent=par[:nn],
                root=root.value)


def test_reference_tree_round_trip(golden):
    from paper_1410_2697_b200.ordering import etree_handle
    g = golden("etree_ref.npz")
    t = foreign_tree(g)
    got = fetch(etree_handle(t))
    for k in ("post", "pptr", "piv", "fptr", "fr", "parent"):
        np.testing.assert_array_equal(got[k], g[k])
    assert got["root"] == int(g["root"])
    assert etree_handle(t) == etree_handle(t)  # flattened once per tree object


def test_reference_tree_equals_native_ordering(golden):
    """The native ND + etree at the same leaf size is the reference's tree."""
    import paper_1410_2697_b200 as P
    g = golden("etree_ref.npz")
    A, _ = P.gen_poisson7(12, 11, 10)
    et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 40), A)
    got = fetch(et._h)
    for k in ("post", "pptr", "piv", "fptr", "fr", "parent"):
        np.testing.assert_array_equal(got[k], g[k])


def _broken(g, **kw):
    t = foreign_tree(g)
    for k, f in kw.items():
        f(t)
    return t


def test_validation_messages(golden):
    from paper_1410_2697_b200.ordering import etree_handle
    g = golden("etree_ref.npz")

    def bad_perm(t):
        t.permutation = np.array(t.permutation).copy()
        t.permutation[0] = t.permutation[1]

    with pytest.raises(ValueError, match="not a permutation"):
        etree_handle(_broken(g, p=bad_perm))

    leaf = int(next(p for p in g["post"] if g["pptr"][p + 1] - g["pptr"][p] >= 3))

    def gap(t):
        nd = t.nodes[leaf]
        nd.pivot_ids = np.concatenate([nd.pivot_ids[:1], nd.pivot_ids[2:]])

    with pytest.raises(ValueError, match="contiguous run"):
        etree_handle(_broken(g, p=gap))

    node = int(next(p for p in g["post"] if g["fptr"][p + 1] > g["fptr"][p] and g["pptr"][p + 1] > g["pptr"][p]))

    def low(t):
        nd = t.nodes[node]
        nd.frontal_ids = np.concatenate([[int(nd.pivot_ids[-1])], nd.frontal_ids])

    # the reference's own RuntimeError text (ordering.py:303-306)
    with pytest.raises(RuntimeError, match=f"node {node}: frontal index below the pivot block"):
        etree_handle(_broken(g, p=low))

    def post_swap(t):
        t.post_order = list(reversed(t.post_order))

    with pytest.raises(ValueError, match="before its child"):
        etree_handle(_broken(g, p=post_swap))


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not mounted (GPU box)")
def test_live_reference_tree_object():
    """The reference's EliminationTree object itself goes through the boundary."""
    import importlib
    import sys
    from paper_1410_2697_b200.ordering import etree_handle
    import paper_1410_2697_b200 as P
    sys.path.insert(0, REFERENCE_SRC)
    try:
        mh = importlib.import_module("mfhodlr")
    finally:
        sys.path.remove(REFERENCE_SRC)
    A, _ = P.gen_poisson7(9, 10, 11)
    R = mh.SparseMatrix(A._csc.copy(), symmetric=True)
    rt = mh.build_elimination_tree(mh.nested_dissection(mh.adjacency_graph(R), 24), R)
    ours = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 24), A)
    a, b = fetch(etree_handle(rt)), fetch(ours._h)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])


@pytest.mark.gpu
def test_factorize_on_the_callers_tree(golden):
    """mf_factorize on the reference's tree (leaf 40): bitwise the same as on
    the native tree of that leaf size, within 1e-8 of the reference's own
    mf_solve, and conventional mode on it solves the system."""
    import paper_1410_2697_b200 as P
    g = golden("etree_ref.npz")
    A, _ = P.gen_poisson7(12, 11, 10)
    kw = dict(n_c=60, eps=1e-6, d=2, n_leaf=16)
    t = foreign_tree(g)
    F = P.mf_factorize(A, t, P.ACCELERATED, P.MfParams(**kw))
    x = P.mf_solve(F, g["b"])
    et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 40), A)
    x2 = P.mf_solve(P.mf_factorize(A, et, P.ACCELERATED, P.MfParams(**kw)), g["b"])
    np.testing.assert_array_equal(x, x2)
    assert F.stats.structured_fronts == int(g["structured"]) and F.stats.peak_stored_reals == int(g["peak"])
    assert np.linalg.norm(x - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])
    xc = P.mf_solve(P.mf_factorize(A, t, P.CONVENTIONAL), g["b"])
    assert np.linalg.norm(xc - g["x_conv"]) <= 1e-10 * np.linalg.norm(g["x_conv"])


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not mounted (GPU box)")
def test_integration_md_binding_builds_the_reference_tree():
    """INTEGRATION.md section 2's _etree_handle, executed as written (minus the
    GPU context), on a live reference EliminationTree."""
    import importlib
    import sys
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    src = open(os.path.join(root, "INTEGRATION.md")).read()
    code = src[src.index("```python\n# mfhodlr/_gpu.py") + 10:]
    code = code[:code.index("```")]
    code = code.replace('C.CDLL("libmfh.so")', repr(os.path.join(root, "paper_1410_2697_b200", "libmfh.so")).join(
        ("C.CDLL(", ")")))
    code = code.replace("_ctx = C.c_void_p(); _check(_L.mfh_ctx_create(0, C.byref(_ctx)))", "_ctx = None")
    ns = {}
    exec(code, ns)
    sys.path.insert(0, REFERENCE_SRC)
    try:
        mh = importlib.import_module("mfhodlr")
    finally:
        sys.path.remove(REFERENCE_SRC)
    import paper_1410_2697_b200 as P
    A, _ = P.gen_poisson7(9, 8, 7)
    R = mh.SparseMatrix(A._csc.copy(), symmetric=True)
    rt = mh.build_elimination_tree(mh.nested_dissection(mh.adjacency_graph(R), 24), R)
    h = ns["_etree_handle"](rt)
    ours = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 24), A)
    a, b = fetch(C.c_void_p(h.value)), fetch(ours._h)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])
