"""Config-scale golden fixtures: the REFERENCE run at BASELINE.json configs[0]
(C1, 2D Q1 128^2) and configs[1] (C2, 3D 7-point 48^3) with the bench's
parameters and seeded right-hand sides.

Run in the build container (where /root/reference is mounted), preferably with
the reference's compiled Cython kernels built in a scratch copy:

    cp -r /root/reference/pkg /tmp/refbuild && (cd /tmp/refbuild && python setup.py build_ext --inplace)
    MFH_REF_SRC=/tmp/refbuild/src OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_configs.py

Per config it stores (tests/golden/cfg_<name>.npz):
  blk        per compressed block, in the reference's visiting order: |I|, |J|, rank
  blkperm    the complete-pivot sequences row_perm[:rank], col_perm[:rank] concatenated
  records    FrontRecord rows (node_id, front_size, n_pivot, path, max_offdiag_rank, stored_reals)
  counters   peak_stored_reals, structured_fronts, dense_fronts, full_square_allocs, stored_reals
  b, x       the seeded RHS and mf_solve(F, b)
  gmres_*    GMRES(restart) to tol: history, iterations, converged, x
  env_*      the reference's own rounding envelope: the same factorization with
             every dense solve inside it (lu_solve / solve_triangular) moved by
             one ulp: relative change of mf_solve, the fraction of blocks whose
             (rank, pivot sequence) stays identical, how many front records and
             which counters move
Large float vectors are stored as float64 (the 1e-8 apply bar needs them);
pivot sequences as int32.
"""

import os
import sys
import time

import numpy as np

REF = os.environ.get("MFH_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import mfhodlr as mh  # noqa: E402
import mfhodlr.bdlr as mbdlr  # noqa: E402
import mfhodlr.hodlr as mhodlr  # noqa: E402
import mfhodlr.multifrontal as mmf  # noqa: E402

from paper_1410_2697_b200 import problems  # noqa: E402  (input generators only)

# name: generator, ND leaf, MfParams, rhs distribution, (tol, restart)  -- bench.py CONFIGS
CASES = {
    "c1": (lambda: problems.gen_q1_2d(128), 64, dict(n_c=256, eps=1e-6, d=1, n_leaf=32), "uniform", (1e-10, 30)),
    "c2": (lambda: problems.gen_poisson7(48, 48, 48), 64, dict(n_c=1024, eps=1e-5, d=1, n_leaf=64), "normal",
           (1e-10, 30)),
}


def factor_with_log(R, tree, params, perturb=False):
    blocks = []
    orig_fplu = mbdlr.full_pivot_lu

    def spy(core, eps, cap):
        res = orig_fplu(core, eps, cap)
        blocks.append((core.shape[0], core.shape[1], res[3], res[1][:res[3]].copy(), res[2][:res[3]].copy()))
        return res

    saved = (mhodlr.lu_solve, mmf.lu_solve, mbdlr.solve_triangular)
    if perturb:
        def up(f):
            return lambda *a, **k: np.nextafter(f(*a, **k), np.inf)
        mhodlr.lu_solve, mmf.lu_solve, mbdlr.solve_triangular = (up(f) for f in saved)
    mbdlr.full_pivot_lu = spy
    try:
        F = mh.mf_factorize(R, tree, mh.ACCELERATED, mh.MfParams(**params))
    finally:
        mbdlr.full_pivot_lu = orig_fplu
        mhodlr.lu_solve, mmf.lu_solve, mbdlr.solve_triangular = saved
    return F, blocks


def run(name):
    gen, leaf, params, dist, (tol, restart) = CASES[name]
    A, _ = gen()
    R = mh.SparseMatrix(A._csc.copy(), symmetric=A.symmetric)
    t0 = time.perf_counter()
    tree = mh.build_elimination_tree(mh.nested_dissection(mh.adjacency_graph(R), leaf), R)
    t1 = time.perf_counter()
    F, blocks = factor_with_log(R, tree, params)
    t2 = time.perf_counter()
    b = problems.seeded_rhs(A.n_rows, 0, dist)
    x = mh.mf_solve(F, b)
    M = mh.Preconditioner(lambda v: mh.mf_solve(F, v), "accelerated-mf")
    xg, h = mh.gmres(mh.LinearOperator.from_matrix(R), b, M=M, tol=tol, restart=restart)
    t3 = time.perf_counter()
    out = {}
    out["blk"] = np.array([[m, n, r] for m, n, r, _, _ in blocks], dtype=np.int32).reshape(-1, 3)
    out["blkperm"] = (np.concatenate([np.stack([rp, cp], 1) for _, _, _, rp, cp in blocks]).astype(np.int32)
                      if blocks else np.zeros((0, 2), np.int32))
    out["records"] = np.array([[r.node_id, r.front_size, r.n_pivot, {"empty": 0, "dense": 1, "structured": 2}[r.path],
                                r.max_offdiag_rank, r.stored_reals] for r in F.stats.records], dtype=np.int64)
    out["counters"] = np.array([F.stats.peak_stored_reals, F.stats.structured_fronts, F.stats.dense_fronts,
                                F.stats.full_square_allocs, F.stored_reals()], dtype=np.int64)
    out["b"] = b
    out["x"] = x
    out["gmres_x"] = xg
    out["gmres_hist"] = np.array(h.residuals)
    out["gmres_meta"] = np.array([h.iterations, int(h.converged), tol, restart])
    out["true_res"] = np.array(np.linalg.norm(A._csc @ xg - b) / np.linalg.norm(b))
    # the reference's own envelope: 1-ulp perturbed dense solves in the factorization
    Fp, bp = factor_with_log(R, tree, params, perturb=True)
    xp = mh.mf_solve(Fp, b)
    same = sum(1 for u, v in zip(blocks, bp) if u[2] == v[2] and np.array_equal(u[3], v[3])
               and np.array_equal(u[4], v[4]))
    out["env_rel"] = np.array(np.linalg.norm(xp - x) / np.linalg.norm(x))
    out["env_pivot_rate"] = np.array(same / max(1, len(blocks)))
    out["env_nblocks"] = np.array([len(blocks), len(bp)])
    # how the reference's own FactorStats move under that perturbation (ranks shift)
    prec = np.array([[r.node_id, r.front_size, r.n_pivot, r.max_offdiag_rank, r.stored_reals]
                     for r in Fp.stats.records], dtype=np.int64)
    out["env_records_mismatch"] = np.array(int(np.sum(np.any(prec != out["records"][:, [0, 1, 2, 4, 5]], axis=1))))
    out["env_counters"] = np.array([Fp.stats.peak_stored_reals, Fp.stats.structured_fronts, Fp.stats.dense_fronts,
                                    Fp.stats.full_square_allocs, Fp.stored_reals()], dtype=np.int64)
    out["timing"] = np.array([t1 - t0, t2 - t1, t3 - t2])
    np.savez_compressed(os.path.join(HERE, f"cfg_{name}.npz"), **out)
    print(f"{name}: backend {mh.KERNEL_BACKEND} blocks {len(blocks)} struct {F.stats.structured_fronts} "
          f"gmres {h.iterations} conv {h.converged} res {h.residuals[-1]:.3e} envelope {float(out['env_rel']):.3e} "
          f"pivot-rate {float(out['env_pivot_rate']):.4f} records-moved {int(out['env_records_mismatch'])} times order {t1 - t0:.1f} factor {t2 - t1:.1f} "
          f"solve {t3 - t2:.1f} s", flush=True)


if __name__ == "__main__":
    for nm in (sys.argv[1:] or sorted(CASES)):
        run(nm)
