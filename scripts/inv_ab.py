"""A/B helper: dump M^{-1} b of the acc_hex_8 golden config to a .npy (bitwise comparisons between kernel variants)."""
import sys
import numpy as np
import paper_1410_2697_b200 as P
from paper_1410_2697_b200 import problems as PR

A, _ = PR.gen_hex_q1(8, seed=3)
et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 32), A)
F = P.mf_factorize(A, et, P.ACCELERATED, P.MfParams(n_c=96, eps=1e-4, d=1, n_leaf=32))
b = np.random.default_rng(0).standard_normal(A.n_rows)
x = P.mf_solve(F, b)
np.save(sys.argv[1], x)
print("ranks", [r.rank for r in F.stats.records][:0], F.stats.structured_fronts, F.stats.peak_stored_reals)
