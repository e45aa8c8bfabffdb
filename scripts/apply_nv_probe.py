"""Device apply time for 1 vs several right-hand sides per replay (development helper)."""
import ctypes as C
import sys
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_1410_2697_b200 as P
from paper_1410_2697_b200 import _lib

side = int(sys.argv[1]) if len(sys.argv) > 1 else 48
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
A, _ = P.gen_poisson7(side, side, side)
et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 64), A)
F = P.mf_factorize(A, et, P.ACCELERATED, P.MfParams(n_c=nc, eps=1e-5 if nc == 1024 else 1e-4, d=1 if nc == 1024 else 2, n_leaf=64))
n = A.n_rows
ctx = _lib.context()
s = torch.cuda.ExternalStream(ctx.info()[0])
B = torch.randn(8, n, dtype=torch.float64, device="cuda")
X = torch.zeros_like(B)
L = _lib.lib()
for nv in (1, 2, 4, 8):
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(5):
                _lib.check(L.mfh_apply(F._h, C.c_void_p(B.data_ptr()), C.c_void_p(X.data_ptr()), nv, 1))
            e1.record(s)
        e1.synchronize()
        if rep == 2:
            print(f"nv {nv}: {e0.elapsed_time(e1) / 5:.3f} ms per replay ({e0.elapsed_time(e1) / 5 / nv:.3f} ms per vector)")
