"""One preconditioner apply (mf_solve) of the C2 factor between cudaProfilerStart/Stop,
for `ncu --profile-from-start off` launch lists of the apply graph (development helper).
Also prints the apply plan's per-level shape (MFH_APPLY_TRACE)."""
import sys
import time
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_1410_2697_b200 as P

side = int(sys.argv[1]) if len(sys.argv) > 1 else 48
A, _ = P.gen_poisson7(side, side, side)
b = P.seeded_rhs(A.n_rows, 0)
et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 64), A)
F = P.mf_factorize(A, et, P.ACCELERATED, P.MfParams(n_c=1024, eps=1e-5, d=1, n_leaf=64))
x = P.mf_solve(F, b)
torch.cuda.synchronize()
for _ in range(3):
    t = time.perf_counter()
    for _ in range(20):
        x = P.mf_solve(F, b)
    print("mf_solve host-array %.3f ms" % ((time.perf_counter() - t) / 20 * 1e3))
for _ in range(3):
    ms, by = F.apply_bench(50)
    print("apply graph replay %.1f us (%.0f GB/s)" % (ms * 1e3, by / ms / 1e6))
torch.cuda.cudart().cudaProfilerStart()
x = P.mf_solve(F, b)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
