"""Repeated factorizations (development helper) to shake out memory-reuse bugs."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1410_2697_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
if cfg == "c2":
    A, _ = P.gen_poisson7(48, 48, 48); kw = dict(n_c=1024, eps=1e-5, d=1, n_leaf=64)
elif cfg == "p32":
    A, _ = P.gen_poisson7(32, 32, 32); kw = dict(n_c=256, eps=1e-5, d=1, n_leaf=64)
else:
    A, _ = P.gen_poisson7(20, 20, 20); kw = dict(n_c=200, eps=1e-5, d=1, n_leaf=64)
b = P.seeded_rhs(A.n_rows, 0)
et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 64), A)
ref = None
keep = []
for r in range(reps):
    F = P.mf_factorize(A, et, P.ACCELERATED, P.MfParams(**kw))
    x = P.mf_solve(F, b)
    if ref is None:
        ref = x
    print(r, "ok", np.linalg.norm(x - ref) / np.linalg.norm(ref), flush=True)
    if r % 3 == 0:
        keep.append(F)   # vary which factors stay alive so pooled chunks get reused in different orders
    if len(keep) > 2:
        keep.pop(0)
