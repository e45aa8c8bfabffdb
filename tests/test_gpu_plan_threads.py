"""BDLR selections on several host threads (plan_front: the blocks of a structured
front are selected concurrently, each thread with its own marker arrays). The
selections are integer and independent, so the factorization must not depend on
the thread count: one thread against eight threads forced onto a small problem
(MFH_PLAN_MIN_EDGES=1 removes the work threshold), with d = 1 (neighbour scan)
and d = 2 (breadth-first search), in separate processes."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_1410_2697_b200 as P
out = {}
for d in (1, 2):
    A, _ = P.gen_poisson7(18, 17, 16)
    et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 32), A)
    F = P.mf_factorize(A, et, P.ACCELERATED, P.MfParams(n_c=64, eps=1e-4, d=d, n_leaf=16))
    x = P.mf_solve(F, P.seeded_rhs(A.n_rows, 3))
    out[str(d)] = {"x": x.tobytes().hex(), "structured": F.stats.structured_fronts,
                   "peak": int(F.stats.peak_stored_reals),
                   "blocks": [[int(v) for v in b.values() if isinstance(v, (int, np.integer))] for b in F.block_log()]}
print(json.dumps(out))
"""


def run(threads, min_edges):
    env = dict(os.environ, MFH_PLAN_THREADS=str(threads), MFH_PLAN_MIN_EDGES=str(min_edges))
    out = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_selection_threads_do_not_change_the_factorization():
    one, eight = run(1, 2e6), run(8, 1)
    for d in ("1", "2"):
        assert one[d]["structured"] > 2
        assert one[d]["blocks"] == eight[d]["blocks"]
        assert one[d]["peak"] == eight[d]["peak"]
        assert one[d]["x"] == eight[d]["x"]
