"""Wall time of the factorization's explicit-inverse dispatch (run_inverse via
mfh_test_inverse_batched) for a batch of B diagonally dominant n x n blocks;
the n = 2 call measures the fixed cost (copies, launch, sync)."""
import os
import sys
import time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_2697_b200 as P  # noqa: F401
from paper_1410_2697_b200 import _lib


def call(n, B, reps=20):
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
    err = np.abs(buf.reshape(B, n, n)[0] @ blocks[0] - np.eye(n)).max()
    return best, err


base, _ = call(2, 1)
print(f"fixed cost {base * 1e6:.1f} us")
for n, B in ((16, 1), (32, 1), (64, 1), (96, 1), (128, 1), (64, 148), (128, 148), (64, 600), (128, 600), (200, 1),
             (316, 1), (316, 8)):
    t, err = call(n, B)
    print(f"n {n:4d} batch {B:4d}: {(t - base) * 1e6:9.1f} us  ({(t - base) * 1e6 / n:6.2f} us/step)  err {err:.1e}",
          flush=True)
