"""Native host symbolic analysis (csrc/symbolic.cpp): adjacency, nested
dissection and elimination tree must be bit-identical to the reference
(golden fixtures) and to the oracle. CPU only — no GPU needed."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_1410_2697_b200 as P
from paper_1410_2697_b200 import problems as PR
from test_oracle import GENS


def native_tree(A, leaf):
    g = P.adjacency_graph(A)
    st = P.nested_dissection(g, leaf)
    return st, P.build_elimination_tree(st, A)


@pytest.mark.parametrize("name", sorted(GENS))
def test_native_ordering_matches_reference_golden(golden, name):
    g = golden("ordering.npz")
    A, _ = GENS[name]()
    leaf = int(g[f"{name}_leaf"])
    st, et = native_tree(A, leaf)
    np.testing.assert_array_equal(st.permutation, g[f"{name}_perm"])
    np.testing.assert_array_equal(np.array(et.post_order), g[f"{name}_post"])
    pp, fp = g[f"{name}_pivptr"], g[f"{name}_frptr"]
    for v in range(len(pp) - 1):
        np.testing.assert_array_equal(et.nodes[v].pivot_ids, g[f"{name}_piv"][pp[v]:pp[v + 1]])
        np.testing.assert_array_equal(et.nodes[v].frontal_ids, g[f"{name}_fr"][fp[v]:fp[v + 1]])


@pytest.mark.parametrize("leaf", [1, 3, 8, 64, 500])
def test_native_matches_oracle_random_sparse(oracle, leaf):
    rng = np.random.default_rng(leaf)
    n = 300
    dense = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.01)
    dense = dense + dense.T + np.diag(np.abs(dense).sum(1) + 1.0)
    A = P.SparseMatrix(sp.csc_matrix(dense))
    st, et = native_tree(A, leaf)
    ip, ix = oracle.adjacency(A._csc)
    g = P.adjacency_graph(A)
    np.testing.assert_array_equal(g.indptr, ip)
    np.testing.assert_array_equal(g.indices, ix)
    ost = oracle.nested_dissection(ip, ix, n, leaf)
    np.testing.assert_array_equal(st.permutation, ost.permutation)
    oet = oracle.build_elimination_tree(ost, A._csc)
    assert oet.post_order == et.post_order
    for v in et.post_order:
        np.testing.assert_array_equal(et.nodes[v].pivot_ids, oet.pivots[v])
        np.testing.assert_array_equal(et.nodes[v].frontal_ids, oet.frontal[v])


def path_graph(n):
    return P.AdjGraph.from_pattern(sp.diags([1.0, 1.0], [-1, 1], shape=(n, n)).tocsr())


def test_path7_leaf3():  # reference tests/test_ordering.py KAT
    tree = P.nested_dissection(path_graph(7), leaf_size=3)
    root = tree.nodes[tree.root]
    assert set(root.vertices.tolist()) == {3}
    kids = {frozenset(tree.nodes[c].vertices.tolist()) for c in root.children}
    assert kids == {frozenset({0, 1, 2}), frozenset({4, 5, 6})}


def test_complete_graph_single_leaf():
    tree = P.nested_dissection(P.AdjGraph.from_pattern(sp.csr_matrix(np.ones((4, 4)))), leaf_size=4)
    assert len(tree.nodes) == 1 and tree.nodes[tree.root].is_leaf


def test_disconnected_components_make_merge_nodes(oracle):
    blocks = sp.block_diag([sp.diags([-1.0, 4.0, -1.0], [-1, 0, 1], shape=(20, 20))] * 3).tocsc()
    A = P.SparseMatrix(blocks, symmetric=True)
    st, et = native_tree(A, 8)
    merges = [v for v in range(len(st.nodes)) if st.nodes[v].children is not None and len(st.nodes[v].vertices) == 0]
    assert merges, "components split under empty-separator nodes (ordering.py:192-197)"
    ost = oracle.nested_dissection(*oracle.adjacency(A._csc), 60, 8)
    np.testing.assert_array_equal(st.permutation, ost.permutation)


def test_explicit_zeros_and_cancellation(oracle):
    # explicit zeros drop out of the ND graph; a_ij + a_ji == 0 drops out of the etree pattern
    d = np.diag(np.full(6, 4.0))
    d[0, 1], d[1, 0] = 1.0, -1.0
    d[2, 3] = 1.0
    A = P.SparseMatrix(sp.csc_matrix(d))
    csc = A._csc.copy()
    csc[4, 5] = 0.0  # explicit zero entry
    A2 = P.SparseMatrix(csc)
    for M in (A, A2):
        st, et = native_tree(M, 1)
        ost = oracle.nested_dissection(*oracle.adjacency(M._csc), 6, 1)
        np.testing.assert_array_equal(st.permutation, ost.permutation)
        oet = oracle.build_elimination_tree(ost, M._csc)
        for v in et.post_order:
            np.testing.assert_array_equal(et.nodes[v].frontal_ids, oet.frontal[v])


def test_validation():
    with pytest.raises(ValueError, match="leaf_size"):
        P.nested_dissection(path_graph(4), leaf_size=0)
    A, _ = PR.gen_poisson7(2, 2, 2)
    st = P.nested_dissection(P.adjacency_graph(A), 4)
    B, _ = PR.gen_poisson7(3, 2, 2)
    with pytest.raises(ValueError, match="does not match"):
        P.build_elimination_tree(st, B)


def test_single_vertex_and_identity():
    A = P.SparseMatrix(sp.eye(1).tocsc(), symmetric=True)
    st, et = native_tree(A, 4)
    assert len(et.nodes) == 1 and et.nodes[0].n_pivot == 1
    A = P.SparseMatrix(sp.eye(10).tocsc(), symmetric=True)
    st, et = native_tree(A, 4)
    assert sorted(st.permutation.tolist()) == list(range(10))
