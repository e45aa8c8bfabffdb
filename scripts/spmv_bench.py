"""SpMV GB/s at the configs' matrices (algorithmic bytes 12 nnz + 4 (N + 1) + 16 N)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1410_2697_b200 as P  # noqa: E402
from paper_1410_2697_b200 import _lib  # noqa: E402

hbm = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6530.3) if os.path.exists("MEASURED_PEAKS.json") else 6530.3
mats = {"c2 7pt 48^3": lambda: P.gen_poisson7(48, 48, 48)[0], "c5 7pt 128^3": lambda: P.gen_poisson7(128, 128, 128)[0]}
if len(sys.argv) > 1 and sys.argv[1] == "all":
    mats["c3 q1 hex 64^3"] = lambda: P.gen_hex_q1(64)[0]
    mats["c4 p1 delaunay 1000^2"] = lambda: P.gen_p1_delaunay(1000)[0]
for name, mk in mats.items():
    A = mk()
    if A is None:
        continue
    op = A.device_operator()
    ms = C.c_double()
    _lib.check(_lib.lib().mfh_spmv_bench(op.handle, 200, C.byref(ms)))
    b = 12.0 * A.nnz + 4.0 * (A.n_rows + 1) + 16.0 * A.n_rows
    x = np.random.default_rng(0).standard_normal(A.n_cols)
    exact = bool(np.array_equal(P.spmv(A, x), A._csc @ x))
    print(f"{name}: {ms.value * 1e3:.1f} us  {b / ms.value / 1e6:.0f} GB/s  frac {b / ms.value / 1e6 / hbm:.3f}  bit-exact {exact}"
          f"  stream={'off' if os.environ.get('MFH_SPMV_NO_STREAM') else 'on'}", flush=True)
