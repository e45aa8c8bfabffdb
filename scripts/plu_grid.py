"""Per-step time of the grouped cooperative complete-pivot LU as a function of
the group size G (MFH_PLU_GRID caps the cooperative grid, so a lone grid-class
core runs as one group of G CTAs): one core at two ranks through
mfh_full_pivot_lu_batched, (t220 - t20) / 200 = microseconds per step."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
m, n = int(sys.argv[1]), int(sys.argv[2])
ts = []
for r in (20, 220):
    B = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    timed(B, 1)
    ts.append(timed(B))
print(f"G {os.environ.get('MFH_PLU_GRID', 'all')} {m}x{n}: {(ts[1] - ts[0]) / 200 * 1e6:7.2f} us/step", flush=True)
