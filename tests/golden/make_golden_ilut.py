"""Fixtures for the baseline preconditioners (krylov.py:164-214): the
REFERENCE's ilut factors (_core.pyx:145-269), its ILUT / diagonal applies and
a GMRES+ILUT history, on seeded problems.

    MFH_REF_SRC=/tmp/refbuild/src OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_ilut.py
"""
import os
import sys

import numpy as np

REF = os.environ.get("MFH_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import mfhodlr as mh  # noqa: E402

from paper_1410_2697_b200 import problems  # noqa: E402

CASES = [
    ("p7_8_k1", lambda: problems.gen_poisson7(8, 8, 8), 1, 1e-4),
    ("p7_10_k2", lambda: problems.gen_poisson7(10, 9, 8), 2, 1e-3),
    ("hex_6_k1", lambda: problems.gen_hex_q1(6, seed=2), 1, 1e-4),
    ("q1_20_k3", lambda: problems.gen_q1_2d(20), 3, 1e-2),
    ("p1_15_k1", lambda: problems.gen_p1_delaunay(15, seed=4), 1, 0.0),
]
out = {}
for name, gen, k, tol in CASES:
    A, _ = gen()
    R = mh.SparseMatrix(A._csc.copy(), symmetric=A.symmetric)
    P = mh.ilut(R, k=k, drop_tol=tol)
    lp, li, lv = P.l_parts
    up, ui, uv = P.u_parts
    b = np.random.default_rng(len(name)).standard_normal(A.n_rows)
    out.update({f"{name}_lp": lp, f"{name}_li": li, f"{name}_lv": lv, f"{name}_up": up, f"{name}_ui": ui,
                f"{name}_uv": uv, f"{name}_b": b, f"{name}_x": P.apply_inverse(b),
                f"{name}_meta": np.array([k, tol, P.stored_reals])})
    D = mh.diagonal_preconditioner(R)
    out[f"{name}_xdiag"] = D.apply_inverse(b)
    x, h = mh.gmres(mh.LinearOperator.from_matrix(R), b, M=P, tol=1e-10, restart=30)
    out[f"{name}_gmres_hist"] = np.array(h.residuals)
    out[f"{name}_gmres_x"] = x
    print(name, "lnz", len(lv), "unz", len(uv), "gmres", h.iterations)
np.savez_compressed(os.path.join(HERE, "ilut.npz"), **out)
