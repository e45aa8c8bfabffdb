"""GPU complete-pivot LU (k_full_pivot_lu) against the reference's own outputs:
bit-exact factors, pivot sequences, ranks and ratios on identical inputs
(the reference's tests/test_kernels.py:22-37 pattern, golden cores included)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_fplu_bit_exact_on_golden_cores(golden):
    import paper_1410_2697_b200 as P
    g = golden("fplu.npz")
    cnt = int(g["count"])
    # batched: several eps values -> group by eps
    by_eps = {}
    for k in range(cnt):
        eps = float(g[f"meta{k}"][0])
        by_eps.setdefault(eps, []).append(k)
    for eps, ks in by_eps.items():
        outs = P.full_pivot_lu_batched([g[f"b{k}"] for k in ks], eps,
                                       [int(g[f"meta{k}"][1]) for k in ks])
        for k, (lu, rp, cp, rank, ratio) in zip(ks, outs):
            _, _, r_ref, q_ref = g[f"meta{k}"]
            assert rank == int(r_ref), k
            assert ratio == q_ref, k
            np.testing.assert_array_equal(rp, g[f"rp{k}"])
            np.testing.assert_array_equal(cp, g[f"cp{k}"])
            np.testing.assert_array_equal(lu, g[f"lu{k}"])


def test_fplu_edge_cases():
    import paper_1410_2697_b200 as P
    lu, rp, cp, rank, ratio = P.full_pivot_lu(np.zeros((4, 5)), 1e-8, 4)
    assert rank == 0 and ratio == 0.0
    lu, rp, cp, rank, ratio = P.full_pivot_lu(np.array([[1.0, -1.0], [1.0, 1.0]]), 1e-15, 2)
    assert rank == 2
    lu, rp, cp, rank, ratio = P.full_pivot_lu(np.ones((1, 1)), 0.5, 1)
    assert rank == 1 and ratio == 0.0


def test_fplu_large_random_vs_oracle(oracle):
    import paper_1410_2697_b200 as P
    rng = np.random.default_rng(7)
    blocks, caps = [], []
    for m, n, r in ((300, 280, 40), (517, 129, 129), (64, 900, 30), (1, 700, 1), (700, 1, 1),
                    (400, 350, 60), (700, 700, 20), (1200, 300, 35),  # cluster paths
                    (1300, 1300, 40), (2100, 900, 25)):  # whole-GPU cooperative path
        B = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
        blocks.append(B)
        caps.append(min(m, n))
    outs = P.full_pivot_lu_batched(blocks, 1e-9, caps)
    for B, cap, (lu, rp, cp, rank, ratio) in zip(blocks, caps, outs):
        olu, orp, ocp, orank, oratio = oracle.full_pivot_lu(B, 1e-9, cap)
        assert rank == orank and ratio == oratio
        np.testing.assert_array_equal(rp, orp)
        np.testing.assert_array_equal(cp, ocp)
        np.testing.assert_array_equal(lu, olu)


def test_fplu_concurrent_groups_vs_oracle(oracle):
    """Five whole-GPU-class cores in one call: the cooperative launch splits into
    five CTA groups factoring concurrently (small groups push the tall cores
    into the global-row launch). Bit-exact against the oracle."""
    import paper_1410_2697_b200 as P
    rng = np.random.default_rng(21)
    blocks, caps = [], []
    for m, n, r, cap in ((1800, 1000, 60, 10**9), (1000, 1800, 30, 10**9), (1500, 1500, 50, 10**9),
                         (2400, 700, 20, 10**9), (900, 900, 900, 120)):
        blocks.append(rng.standard_normal((m, r)) @ rng.standard_normal((r, n)))
        caps.append(min(m, n, cap))
    outs = P.full_pivot_lu_batched(blocks, 1e-9, caps)
    for B, cap, (lu, rp, cp, rank, ratio) in zip(blocks, caps, outs):
        olu, orp, ocp, orank, oratio = oracle.full_pivot_lu(B, 1e-9, cap)
        assert rank == orank and ratio == oratio
        np.testing.assert_array_equal(rp, orp)
        np.testing.assert_array_equal(cp, ocp)
        np.testing.assert_array_equal(lu, olu)


def test_spmv_matches_scipy():
    import paper_1410_2697_b200 as P
    A, _ = P.gen_poisson7(20, 17, 13)
    x = np.random.default_rng(0).standard_normal(A.n_rows)
    y = P.spmv(A, x)
    assert np.linalg.norm(y - A._csc @ x) <= 1e-14 * np.linalg.norm(A._csc @ x)
    with pytest.raises(ValueError, match="dimension mismatch"):
        P.spmv(A, np.ones(3))


def test_spmv_streamed_bit_identical_to_reference_product():
    """k_spmv_stream adds each row's rounded products in ascending column order from 0:
    the reference's scipy CSC product (sparse.py:284) bit for bit. Ragged rows, empty rows,
    rows at every 16-byte misalignment of the bulk copies, a chunk tail, many chunks per CTA."""
    import scipy.sparse as sp
    import paper_1410_2697_b200 as P
    rng = np.random.default_rng(5)
    cases = [P.gen_poisson7(20, 17, 13)[0], P.gen_poisson7(64, 64, 40)[0]]
    for n, dens, seed in [(1, 1.0, 0), (257, 0.02, 1), (5000, 0.002, 2), (1031, 0.03, 3), (70000, 0.0001, 4)]:
        g = np.random.default_rng(seed)
        m = max(1, int(dens * n * n))
        M = sp.coo_matrix((np.ones(m), (g.integers(0, n, m), g.integers(0, n, m))), shape=(n, n)).tocsr()
        M.data = g.standard_normal(M.nnz)
        if n > 10:                 # two empty rows
            keep = sp.diags((~np.isin(np.arange(n), [3, n // 2])).astype(np.float64))
            M = keep @ M
            M.eliminate_zeros()
        cases.append(P.SparseMatrix(sp.csc_matrix(M)))
    # no entries at all, and a rectangular matrix
    cases.append(P.SparseMatrix(sp.csc_matrix((5, 5))))
    cases.append(P.SparseMatrix(sp.random(300, 200, density=0.05, random_state=9, format="csc")))
    # rows of 40-200 entries (32-row chunks) and a matrix whose rows are too long to stream (fallback kernel)
    cases.append(P.SparseMatrix(sp.random(600, 600, density=0.2, random_state=7, format="csc")))
    long_rows = P.SparseMatrix(sp.random(900, 900, density=0.6, random_state=8, format="csc"))
    for A in cases:
        x = rng.standard_normal(A.n_cols)
        np.testing.assert_array_equal(P.spmv(A, x), A._csc @ x)
    x = rng.standard_normal(900)
    ref = long_rows._csc @ x
    assert np.linalg.norm(P.spmv(long_rows, x) - ref) <= 1e-14 * np.linalg.norm(ref)


def _gpu_inverse(mats):
    import ctypes as C
    from paper_1410_2697_b200 import _lib
    ns = np.array([m.shape[0] for m in mats], dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(ns * ns)[:-1]]).astype(np.int64)
    buf = np.concatenate([np.ascontiguousarray(m, dtype=np.float64).ravel() for m in mats])
    sing = np.zeros(len(mats), dtype=np.int32)
    ctx = _lib.context()
    _lib.check(_lib.lib().mfh_test_inverse_batched(ctx.handle, len(mats), _lib.ptr(offs), _lib.ptr(ns),
                                                   _lib.ptr(buf), buf.size, _lib.ptr(sing)))
    return [buf[o:o + n * n].reshape(n, n) for o, n in zip(offs, ns)], sing


SIZES = [1, 2, 5, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129, 200, 257, 450, 700, 1000]


def test_explicit_inverse_with_pivoting():
    """Every size class of the factorization's inverse dispatch (64- and
    128-wide register Gauss-Jordan, blocked panel LU + triangular inverses)
    on random non-symmetric blocks, where partial pivoting moves rows from
    every warp/lane position."""
    rng = np.random.default_rng(11)
    mats = [rng.standard_normal((n, n)) for n in SIZES]
    invs, sing = _gpu_inverse(mats)
    assert not sing.any()
    for a, x in zip(mats, invs):
        n = a.shape[0]
        ref = np.linalg.inv(a)
        err = np.abs(x - ref).max() / np.abs(ref).max()
        assert err < 1e-9 * n, (n, err)
        assert np.abs(a @ x - np.eye(n)).max() < 1e-9 * n, n


def test_explicit_inverse_exact_permutations_and_singular():
    """Scaled anti-diagonal permutations pivot on the last row at every step:
    inverses are exact. A zero column is reported singular."""
    mats = []
    for n in (7, 40, 64, 96, 128, 300, 600, 1000):
        p = np.zeros((n, n))
        p[np.arange(n), n - 1 - np.arange(n)] = 2.0 ** (np.arange(n) % 7 - 3)
        mats.append(p)
    z = np.eye(50)
    z[:, 17] = 0.0
    z2 = np.eye(200)
    z2[:, 150] = 0.0
    invs, sing = _gpu_inverse(mats + [z, z2])
    for a, x in zip(mats, invs):
        np.testing.assert_array_equal(x, np.linalg.inv(a))
    assert sing.tolist() == [0] * len(mats) + [1, 1]
