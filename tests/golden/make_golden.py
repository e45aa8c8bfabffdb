"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (where /root/reference is mounted):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference imports with its pure-numpy kernel backend (``_pure``), which its
own tests pin bit-identical to the compiled ``_core`` (tests/test_kernels.py:22-37).
Nothing here is needed at test time: the fixtures are committed .npz files.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import mfhodlr as mh  # noqa: E402
import mfhodlr.bdlr as mbdlr  # noqa: E402
from mfhodlr._kernels import full_pivot_lu as ref_fplu  # noqa: E402

from paper_1410_2697_b200 import problems  # noqa: E402  (input generators only)


def ref_matrix(A):
    """Same matrix as a reference SparseMatrix."""
    return mh.SparseMatrix(A._csc.copy(), symmetric=A.symmetric)


def fplu_cases():
    rng = np.random.default_rng(0)
    out = {}
    blocks = []
    for _ in range(40):
        m = int(rng.integers(1, 40))
        n = int(rng.integers(1, 40))
        r = int(rng.integers(1, min(m, n) + 1))
        B = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
        eps = float(10.0 ** -rng.integers(2, 14))
        cap = int(rng.integers(1, min(m, n) + 1))
        blocks.append((B, eps, cap))
    # ties and integer-valued blocks (Poisson-like) exercise first-max tie-breaking
    for _ in range(20):
        m = int(rng.integers(2, 30))
        n = int(rng.integers(2, 30))
        B = rng.integers(-2, 3, size=(m, n)).astype(float)
        blocks.append((B, 1e-6, min(m, n)))
    blocks.append((np.zeros((4, 5)), 1e-8, 4))
    blocks.append((np.array([[1.0, -1.0], [1.0, 1.0]]), 1e-15, 2))
    # real cores captured from a reference factorization (BDLR pseudoskeletons)
    captured = []
    orig = mbdlr.full_pivot_lu

    def spy(core, eps, cap):
        if len(captured) < 300:
            captured.append((np.array(core, copy=True), float(eps), int(cap)))
        return orig(core, eps, cap)

    mbdlr.full_pivot_lu = spy
    try:
        A, _ = mh.gen_poisson7(12, 12, 12)
        tree = mh.build_elimination_tree(mh.nested_dissection(mh.adjacency_graph(A), 64), A)
        mh.mf_factorize(A, tree, mh.ACCELERATED, mh.MfParams(n_c=64, eps=1e-5, d=1, n_leaf=16))
    finally:
        mbdlr.full_pivot_lu = orig
    blocks += captured[::3]
    for k, (B, eps, cap) in enumerate(blocks):
        lu, rp, cp, rank, ratio = ref_fplu(B, eps, cap)
        out[f"b{k}"] = B
        out[f"lu{k}"] = lu
        out[f"rp{k}"] = rp
        out[f"cp{k}"] = cp
        out[f"meta{k}"] = np.array([eps, cap, rank, ratio])
    out["count"] = np.array(len(blocks))
    np.savez_compressed(os.path.join(HERE, "fplu.npz"), **out)
    print("fplu cases", len(blocks))


ORDER_CASES = [
    ("p7_6", lambda: problems.gen_poisson7(6, 6, 6), 16),
    ("p7_12_11_10", lambda: problems.gen_poisson7(12, 11, 10), 64),
    ("q1_40", lambda: problems.gen_q1_2d(40), 32),
    ("hex_8", lambda: problems.gen_hex_q1(8, seed=3), 32),
    ("p1_30", lambda: problems.gen_p1_delaunay(30, seed=1), 64),
]


def ordering_cases():
    out = {}
    for name, gen, leaf in ORDER_CASES:
        A, _ = gen()
        R = ref_matrix(A)
        st = mh.nested_dissection(mh.adjacency_graph(R), leaf_size=leaf)
        t = mh.build_elimination_tree(st, R)
        nn = len(t.nodes)
        piv_ptr = np.zeros(nn + 1, dtype=np.int64)
        fr_ptr = np.zeros(nn + 1, dtype=np.int64)
        pivs, frs = [], []
        for v in range(nn):
            pivs.append(t.nodes[v].pivot_ids)
            frs.append(t.nodes[v].frontal_ids)
            piv_ptr[v + 1] = piv_ptr[v] + len(t.nodes[v].pivot_ids)
            fr_ptr[v + 1] = fr_ptr[v] + len(t.nodes[v].frontal_ids)
        out[f"{name}_perm"] = t.permutation
        out[f"{name}_post"] = np.array(t.post_order, dtype=np.int64)
        out[f"{name}_pivptr"] = piv_ptr
        out[f"{name}_piv"] = np.concatenate(pivs) if pivs else np.zeros(0, np.int64)
        out[f"{name}_frptr"] = fr_ptr
        out[f"{name}_fr"] = np.concatenate(frs) if frs else np.zeros(0, np.int64)
        out[f"{name}_leaf"] = np.array(leaf)
    np.savez_compressed(os.path.join(HERE, "ordering.npz"), **out)
    print("ordering cases", len(ORDER_CASES))


# (name, generator, ND leaf, mode, params, rhs seed, gmres (tol, restart) or None)
MF_CASES = [
    ("conv_p7_6", lambda: problems.gen_poisson7(6, 6, 6), 16, "conventional", {}, 0, None),
    ("acc_p7_8", lambda: problems.gen_poisson7(8, 8, 8), 16, "accelerated",
     dict(n_c=32, eps=1e-5, d=1, n_leaf=16), 1, (1e-10, 30)),
    ("acc_p7_12", lambda: problems.gen_poisson7(12, 12, 12), 64, "accelerated",
     dict(n_c=64, eps=1e-5, d=1, n_leaf=16), 2, (1e-10, 30)),
    ("acc_p7_10_d2", lambda: problems.gen_poisson7(10, 10, 10), 32, "accelerated",
     dict(n_c=64, eps=1e-3, d=2, n_leaf=32), 3, None),
    ("acc_q1_48", lambda: problems.gen_q1_2d(48), 32, "accelerated",
     dict(n_c=96, eps=1e-6, d=1, n_leaf=32), 4, (1e-10, 30)),
    ("acc_p7_16", lambda: problems.gen_poisson7(16, 16, 16), 64, "accelerated",
     dict(n_c=256, eps=1e-5, d=1, n_leaf=64), 5, (1e-10, 30)),
    ("acc_p7_8_tight", lambda: problems.gen_poisson7(8, 8, 8), 64, "accelerated",
     dict(n_c=32, eps=1e-12, d=3, n_leaf=64), 6, None),
    ("acc_hex_8", lambda: problems.gen_hex_q1(8, seed=3), 32, "accelerated",
     dict(n_c=96, eps=1e-4, d=1, n_leaf=32), 7, (1e-10, 50)),
    ("acc_p7_12_cap", lambda: problems.gen_poisson7(12, 12, 12), 64, "accelerated",
     dict(n_c=64, eps=1e-8, d=1, n_leaf=16, max_rank=5), 8, None),
]


def mf_cases():
    out = {}
    for name, gen, leaf, mode, kw, seed, gm in MF_CASES:
        A, _ = gen()
        R = ref_matrix(A)
        tree = mh.build_elimination_tree(mh.nested_dissection(mh.adjacency_graph(R), leaf), R)
        blocks = []
        orig = mbdlr.full_pivot_lu

        def spy(core, eps, cap):
            res = orig(core, eps, cap)
            blocks.append((core.shape[0], core.shape[1], res[3], res[1][:res[3]].copy(),
                           res[2][:res[3]].copy()))
            return res

        mbdlr.full_pivot_lu = spy
        try:
            F = mh.mf_factorize(R, tree, mode, mh.MfParams(**kw) if kw else None)
        finally:
            mbdlr.full_pivot_lu = orig
        b = np.random.default_rng(seed).standard_normal(A.n_rows)
        x = mh.mf_solve(F, b)
        recs = np.array([[r.node_id, r.front_size, r.n_pivot, {"empty": 0, "dense": 1, "structured": 2}[r.path],
                          r.max_offdiag_rank, r.stored_reals] for r in F.stats.records], dtype=np.int64)
        out[f"{name}_b"] = b
        out[f"{name}_x"] = x
        out[f"{name}_records"] = recs
        out[f"{name}_counters"] = np.array([F.stats.peak_stored_reals, F.stats.structured_fronts,
                                            F.stats.dense_fronts, F.stats.full_square_allocs,
                                            F.stored_reals()], dtype=np.int64)
        out[f"{name}_blk"] = np.array([[m, n, r] for m, n, r, _, _ in blocks], dtype=np.int64).reshape(-1, 3)
        out[f"{name}_blkperm"] = (np.concatenate([np.stack([rp, cp], 1) for _, _, _, rp, cp in blocks])
                                  if blocks else np.zeros((0, 2), np.int64))
        if gm is not None:
            tol, restart = gm
            M = mh.Preconditioner(lambda v: mh.mf_solve(F, v), "accelerated-mf")
            xg, h = mh.gmres(mh.LinearOperator.from_matrix(R), b, M=M, tol=tol, restart=restart)
            out[f"{name}_gmres_x"] = xg
            out[f"{name}_gmres_hist"] = np.array(h.residuals)
            out[f"{name}_gmres_meta"] = np.array([h.iterations, int(h.converged), tol, restart])
        print(name, "blocks", len(blocks), "struct", F.stats.structured_fronts)
    np.savez_compressed(os.path.join(HERE, "mf.npz"), **out)


def gmres_cases():
    """Dense-operator GMRES KATs (test_krylov.py style) with the reference outputs."""
    out = {}
    rng = np.random.default_rng(11)
    cases = []
    for n, restart, tol in ((8, 100, 1e-10), (30, 30, 1e-12), (40, 5, 1e-9), (50, 4, 1e-14)):
        A = rng.standard_normal((n, n)) * (0.3 if n == 40 else 1.0) + (n / 4 if n == 40 else (2 if n == 50 else n)) * np.eye(n)
        b = rng.standard_normal(n)
        max_iter = 7 if n == 50 else 4000
        x, h = mh.gmres(mh.LinearOperator.from_matrix(A), b, tol=tol, restart=restart, max_iter=max_iter)
        k = len(cases)
        out[f"A{k}"] = A
        out[f"b{k}"] = b
        out[f"x{k}"] = x
        out[f"hist{k}"] = np.array(h.residuals)
        out[f"meta{k}"] = np.array([restart, tol, max_iter, h.iterations, int(h.converged)])
        cases.append(k)
    out["count"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "gmres.npz"), **out)
    print("gmres cases", len(cases))


if __name__ == "__main__":
    assert mh.KERNEL_BACKEND in ("pure", "compiled")
    fplu_cases()
    ordering_cases()
    mf_cases()
    gmres_cases()
