"""One complete-pivot LU core (for ncu captures of a single kernel class)."""
import sys
import numpy as np
import paper_1410_2697_b200 as P

m, n, r = (int(x) for x in sys.argv[1:4])
rng = np.random.default_rng(0)
B = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
P.full_pivot_lu_batched([B], 1e-14, [min(m, n)])
print("ok", m, n, r)
