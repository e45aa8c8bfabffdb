"""Fixture for the caller-supplied elimination tree (mfh_etree_from_arrays):
the REFERENCE's own EliminationTree at a non-default ND leaf size (40), fully
flattened (permutation, parent, children, post order, pivot / frontal ids),
with the reference's mf_solve on it.

    MFH_REF_SRC=/tmp/refbuild/src OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_etree.py
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

A, _ = problems.gen_poisson7(12, 11, 10)
R = mh.SparseMatrix(A._csc.copy(), symmetric=True)
tree = mh.build_elimination_tree(mh.nested_dissection(mh.adjacency_graph(R), 40), R)
nn = len(tree.nodes)
out = {"perm": np.asarray(tree.permutation, dtype=np.int64), "post": np.asarray(tree.post_order, dtype=np.int64),
       "root": np.array(tree.root)}
parent = np.array([-1 if nd.parent is None else nd.parent for nd in tree.nodes], dtype=np.int64)
cptr, kids, pptr, piv, fptr, fr = [0], [], [0], [], [0], []
for nd in tree.nodes:
    kids += list(nd.children)
    cptr.append(len(kids))
    piv += list(nd.pivot_ids)
    pptr.append(len(piv))
    fr += list(nd.frontal_ids)
    fptr.append(len(fr))
out.update(parent=parent, cptr=np.array(cptr), child=np.array(kids, dtype=np.int64), pptr=np.array(pptr),
           piv=np.array(piv, dtype=np.int64), fptr=np.array(fptr), fr=np.array(fr, dtype=np.int64))
params = dict(n_c=60, eps=1e-6, d=2, n_leaf=16)
F = mh.mf_factorize(R, tree, mh.ACCELERATED, mh.MfParams(**params))
b = np.random.default_rng(17).standard_normal(A.n_rows)
out["b"] = b
out["x"] = mh.mf_solve(F, b)
out["peak"] = np.array(F.stats.peak_stored_reals)
out["structured"] = np.array(F.stats.structured_fronts)
Fc = mh.mf_factorize(R, tree, mh.CONVENTIONAL)
out["x_conv"] = mh.mf_solve(Fc, b)
np.savez_compressed(os.path.join(HERE, "etree_ref.npz"), **out)
print("nodes", nn, "structured", F.stats.structured_fronts, "peak", F.stats.peak_stored_reals)
