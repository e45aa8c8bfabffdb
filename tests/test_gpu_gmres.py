"""GPU GMRES (mfh_gmres) against the reference: dense-operator golden cases
(iteration counts and histories), preconditioned solves (iterations +-1, same
final residual) and the reference's krylov KATs."""
import numpy as np
import pytest

from test_oracle import MF

pytestmark = pytest.mark.gpu


def op(M):
    import paper_1410_2697_b200 as P
    return P.LinearOperator.from_matrix(np.asarray(M, dtype=np.float64))


def test_golden_dense_cases(golden):
    import paper_1410_2697_b200 as P
    g = golden("gmres.npz")
    for k in range(int(g["count"])):
        restart, tol, max_iter, its, conv = g[f"meta{k}"]
        x, h = P.gmres(op(g[f"A{k}"]), g[f"b{k}"], tol=tol, restart=int(restart), max_iter=int(max_iter))
        assert h.iterations == int(its) and h.converged == bool(conv)
        np.testing.assert_allclose(h.residuals, g[f"hist{k}"], rtol=1e-6, atol=1e-14)  # entries ~1e-16 are rounding noise
        np.testing.assert_allclose(x, g[f"x{k}"], rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("name", ["acc_p7_8", "acc_p7_12", "acc_q1_48", "acc_p7_16", "acc_hex_8"])
def test_preconditioned_against_golden(golden, name):
    import paper_1410_2697_b200 as P
    g = golden("mf.npz")
    gen, leaf, mode, kw = MF[name]
    A, _ = gen()
    et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), leaf), A)
    F = P.mf_factorize(A, et, mode, P.MfParams(**kw))
    its, conv, tol, restart = g[f"{name}_gmres_meta"]
    x, h = P.gmres(A, g[f"{name}_b"], M=P.mf_preconditioner(F), tol=tol, restart=int(restart))
    assert h.converged == bool(conv)
    assert abs(h.iterations - int(its)) <= 1
    b = g[f"{name}_b"]
    assert np.linalg.norm(A._csc @ x - b) / np.linalg.norm(b) <= tol


def test_identity_one_iteration():
    import paper_1410_2697_b200 as P
    b = np.array([1.0, -2.0, 0.5])
    x, h = P.gmres(op(np.eye(3)), b, tol=1e-10)
    assert h.converged and h.iterations == 1
    np.testing.assert_allclose(x, b, atol=1e-12)


def test_2x2_hand_solution():
    import paper_1410_2697_b200 as P
    x, h = P.gmres(op([[4.0, 1.0], [1.0, 3.0]]), np.array([1.0, 2.0]), tol=1e-12)
    assert h.converged and h.iterations <= 2
    np.testing.assert_allclose(x, [1 / 11, 7 / 11], atol=1e-10)


def test_exact_preconditioner_callback():
    import paper_1410_2697_b200 as P
    rng = np.random.default_rng(0)
    A = rng.standard_normal((8, 8)) + 8 * np.eye(8)
    inv = np.linalg.inv(A)
    M = P.Preconditioner(lambda v: inv @ v, "accelerated-mf")
    b = rng.standard_normal(8)
    x, h = P.gmres(op(A), b, M=M, tol=1e-10)
    assert h.converged and h.iterations == 1
    np.testing.assert_allclose(A @ x, b, atol=1e-9)


def test_zero_rhs_and_history_invariants():
    import paper_1410_2697_b200 as P
    x, h = P.gmres(op(np.eye(4)), np.zeros(4), tol=1e-8)
    assert h.converged and h.iterations == 0 and h.residuals == [0.0]
    rng = np.random.default_rng(5)
    A = rng.standard_normal((12, 12)) + 12 * np.eye(12)
    _, h = P.gmres(op(A), rng.standard_normal(12), tol=1e-10)
    assert all(r >= 0 for r in h.residuals) and h.residuals[-1] <= 1e-10
    assert len(h.residuals) == h.iterations


def test_callback_operator_nan_raises_and_validation():
    import paper_1410_2697_b200 as P
    bad = P.LinearOperator(2, lambda v: np.array([np.nan, np.nan]))
    with pytest.raises(ValueError, match="not finite"):
        P.gmres(bad, np.ones(2), tol=1e-6)
    with pytest.raises(ValueError, match="tol"):
        P.gmres(op(np.eye(2)), np.ones(2), tol=2.0)
    with pytest.raises(ValueError, match="dimension"):
        P.gmres(op(np.eye(2)), np.ones(3))


def test_max_iter_cap():
    import paper_1410_2697_b200 as P
    rng = np.random.default_rng(6)
    A = rng.standard_normal((50, 50)) + 2 * np.eye(50)
    _, h = P.gmres(op(A), rng.standard_normal(50), tol=1e-14, restart=4, max_iter=7)
    assert h.iterations <= 7 and not h.converged


@pytest.mark.parametrize("restart", [6, 30])
def test_batched_rhs_match_single_solves(restart):
    """gmres_batched (groups of up to eight right-hand sides sharing each
    preconditioner apply on the FP64 tensor cores) against one gmres call per
    column (warp-per-row apply): the same solves to rounding -- iteration
    counts within one, residual histories and solutions to 1e-8 -- across a
    group boundary (10 = 8 + 2), with restarts (restart 6) and a zero column."""
    import paper_1410_2697_b200 as P
    A, _ = P.gen_poisson7(12, 11, 10)
    et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 32), A)
    F = P.mf_factorize(A, et, P.ACCELERATED, P.MfParams(n_c=96, eps=1e-2, n_leaf=16))
    M = P.mf_preconditioner(F)
    B = np.random.default_rng(5).standard_normal((A.n_rows, 10))
    B[:, 3] = 0.0
    X, hs = P.gmres_batched(A, B, M, tol=1e-10, restart=restart)
    for j in range(B.shape[1]):
        x, h = P.gmres(A, B[:, j], M=M, tol=1e-10, restart=restart)
        assert abs(hs[j].iterations - h.iterations) <= 1 and hs[j].converged == h.converged
        n = min(len(hs[j].residuals), len(h.residuals))
        np.testing.assert_allclose(hs[j].residuals[:n - 1], h.residuals[:n - 1], rtol=1e-6, atol=1e-14)
        np.testing.assert_allclose(X[:, j], x, rtol=0, atol=1e-8 * max(1.0, np.abs(x).max()))
    assert hs[0].iterations > restart if restart == 6 else True
