"""Compare device-resident vs host-array GMRES on one factorization (development helper)."""
import ctypes as C, sys, time
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_1410_2697_b200 as P
from paper_1410_2697_b200 import _lib
A, _ = P.gen_poisson7(48, 48, 48)
b = P.seeded_rhs(A.n_rows, 0)
et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 64), A)
ctx = _lib.context()
F = P.mf_factorize(A, et, P.ACCELERATED, P.MfParams(n_c=1024, eps=1e-5, d=1, n_leaf=64))
dev_op = A.device_operator()
n = A.n_rows
d_b = torch.from_numpy(b).cuda(); d_x = torch.zeros(n, dtype=torch.float64, device="cuda")
hist = np.empty(4000)
for rep in range(4):
    ops = _lib.mfh_gmres_ops(); ops.A = dev_op.handle; ops.M = F._h
    nh, its, conv = C.c_int64(), C.c_int64(), C.c_int()
    torch.cuda.synchronize(); t = time.perf_counter()
    _lib.check(_lib.lib().mfh_gmres_device(ctx.handle, C.byref(ops), n, C.c_void_p(d_b.data_ptr()), C.c_void_p(d_x.data_ptr()), 1e-10, 4000, 30, _lib.ptr(hist), C.byref(nh), C.byref(its), C.byref(conv)))
    t1 = time.perf_counter() - t
    torch.cuda.synchronize(); t = time.perf_counter()
    x, h = P.gmres(A, b, M=P.mf_preconditioner(F), tol=1e-10, restart=30)
    t2 = time.perf_counter() - t
    print(f"rep {rep}: device-path {t1*1e3:.1f} ms ({its.value} its), host-path {t2*1e3:.1f} ms ({h.iterations} its), inner {F.timing()['gmres_ms']:.1f}", flush=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(2):
    flush.fill_(1); torch.cuda.synchronize()
    t = time.perf_counter()
    _lib.check(_lib.lib().mfh_gmres_device(ctx.handle, C.byref(ops), n, C.c_void_p(d_b.data_ptr()), C.c_void_p(d_x.data_ptr()), 1e-10, 4000, 30, _lib.ptr(hist), C.byref(nh), C.byref(its), C.byref(conv)))
    print("after flush", (time.perf_counter() - t) * 1e3, flush=True)
