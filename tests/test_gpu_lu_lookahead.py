"""Blocked-LU look-ahead (run_getrf, MFH_LU_LOOKAHEAD_MIN): the next panel is
factored on its own stream beside the rest of the trailing update, which is
split into the next panel's columns and the others. The split only regroups
output tiles and the panel touches columns the rest of the update leaves alone,
so explicit inverses must come out bit for bit the same with the look-ahead on
(threshold 256 rows) and off (the default), in separate processes."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_1410_2697_b200 as P
from paper_1410_2697_b200 import _lib
out = {}
for n, B in ((300, 3), (700, 2), (1500, 1)):
    rng = np.random.default_rng(n)
    blocks = rng.standard_normal((B, n, n))
    buf = blocks.ravel().copy()
    offs = np.arange(B, dtype=np.int64) * n * n
    ns = np.full(B, n, dtype=np.int64)
    sing = np.zeros(B, dtype=np.int32)
    _lib.check(_lib.lib().mfh_test_inverse_batched(_lib.context().handle, B, _lib.ptr(offs), _lib.ptr(ns),
                                                   _lib.ptr(buf), buf.size, _lib.ptr(sing)))
    err = float(np.abs(buf.reshape(B, n, n)[0] @ blocks[0] - np.eye(n)).max())
    out[str(n)] = {"sha": hashlib.sha256(buf.tobytes()).hexdigest(), "err": err, "sing": sing.tolist()}
print(json.dumps(out))
"""


def run(env_extra):
    env = dict(os.environ)
    env.pop("MFH_LU_LOOKAHEAD_MIN", None)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_lookahead_inverses_bitwise():
    off, on = run({}), run({"MFH_LU_LOOKAHEAD_MIN": "256"})
    for n in ("300", "700", "1500"):
        assert off[n]["sing"] == on[n]["sing"] and not any(off[n]["sing"])
        assert off[n]["err"] < 1e-6
        assert off[n]["sha"] == on[n]["sha"]
