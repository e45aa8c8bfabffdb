"""Materialized child updates (MFH_DENSIFY_MIN): the parent's extend-add reads a
dense copy of a large child update (update HODLR - W V^T formed by k_gemm)
instead of evaluating it per sampled entry. Both forms use the same
k-ascending FMA chains and the same final subtraction, so the factorization
must be bitwise the same; checked in two processes (the threshold is read once
per process) on a problem with structured children."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_1410_2697_b200 as P
A, _ = P.gen_poisson7(18, 17, 16)
et = P.build_elimination_tree(P.nested_dissection(P.adjacency_graph(A), 32), A)
F = P.mf_factorize(A, et, P.ACCELERATED, P.MfParams(n_c=64, eps=1e-4, d=1, n_leaf=16))
b = P.seeded_rhs(A.n_rows, 3)
x = P.mf_solve(F, b)
print(json.dumps({"x": x.tobytes().hex(), "structured": F.stats.structured_fronts,
                  "blocks": [[int(v) for v in d.values() if isinstance(v, (int, np.integer))] for d in F.block_log()]}))
"""


def run(threshold):
    env = dict(os.environ, MFH_DENSIFY_MIN=str(threshold))
    out = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_densified_updates_bitwise():
    a, b = run(0), run(64)
    assert a["structured"] > 2
    assert a["blocks"] == b["blocks"]
    assert a["x"] == b["x"]
