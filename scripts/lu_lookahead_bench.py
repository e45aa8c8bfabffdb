"""Explicit inverse (blocked LU + triangular inverses) of large blocks through
mfh_test_inverse_batched: wall time including the host copies (identical for
both settings), MFH_LU_LOOKAHEAD_MIN on / off in separate processes."""
import os
import sys
import time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_2697_b200 as P  # noqa: F401
from paper_1410_2697_b200 import _lib


def call(n, B, reps=4):
    rng = np.random.default_rng(0)
    blocks = rng.standard_normal((B, n, n)) + 2 * n * np.eye(n)
    flat = np.ascontiguousarray(blocks.ravel())
    offs = np.arange(B, dtype=np.int64) * n * n
    ns = np.full(B, n, dtype=np.int64)
    sing = np.zeros(B, dtype=np.int32)
    best = 1e9
    for _ in range(reps):
        buf = flat.copy()
        t = time.perf_counter()
        _lib.check(_lib.lib().mfh_test_inverse_batched(_lib.context().handle, B, _lib.ptr(offs), _lib.ptr(ns),
                                                       _lib.ptr(buf), buf.size, _lib.ptr(sing)))
        best = min(best, time.perf_counter() - t)
    return best, buf


tag = "off" if os.environ.get("MFH_LU_LOOKAHEAD_MIN") else "on"
for n, B in ((1024, 1), (2048, 1), (4096, 1), (8192, 1), (4096, 4), (2048, 16)):
    t, buf = call(n, B)
    np.save(f"/tmp/inv_{tag}_{n}_{B}.npy", buf[: n * n])
    print(f"lookahead {tag} n {n:5d} batch {B:3d}: {t * 1e3:9.2f} ms", flush=True)
    other = f"/tmp/inv_{'on' if tag == 'off' else 'off'}_{n}_{B}.npy"
    if os.path.exists(other):
        print("   bitwise equal to the other setting:", bool(np.array_equal(np.load(other), buf[: n * n])))
