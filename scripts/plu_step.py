"""Per-step cost of the complete-pivot LU kernel classes: time one core of a
given size at two ranks through mfh_full_pivot_lu_batched (copies cancel in the
difference) -> microseconds per elimination step.

Caveat: the call includes pageable host copies of the core; for cores above
~1M entries their run-to-run variance is of the order of the difference, so
use the bench's device-timed pivot-LU phase for decisions at those sizes."""
import time
import numpy as np
import torch
import paper_1410_2697_b200 as P


def timed(B, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        P.full_pivot_lu_batched([B], 1e-14, [min(B.shape)])
        best = min(best, time.perf_counter() - t)
    return best


rng = np.random.default_rng(0)
for m, n in ((100, 120), (180, 300), (300, 300), (600, 600), (1000, 1000), (1728, 971)):
    ts = []
    for r in (20, 220):
        B = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
        timed(B, 1)
        ts.append(timed(B))
    print(f"{m}x{n}: {(ts[1] - ts[0]) / 200 * 1e6:7.2f} us/step  (t20 {ts[0]*1e3:.2f} ms, t220 {ts[1]*1e3:.2f} ms)",
          flush=True)
