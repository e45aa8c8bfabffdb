"""The apply's batched GEMV against host references of the kernels' own
arithmetic, bit for bit.

One right-hand side (k_gemv2, a warp per row): lane l sums the columns
k = l (mod 32) as a k-ascending chain of correctly rounded FMAs, the 32 lane
sums meet in a shuffle-down tree (lane l += lane l + o for o = 16, 8, 4, 2, 1).

Several right-hand sides (k_gemv_tc: rows in groups of 8 on the FP64 tensor
cores, mma.sync m8n8k4, 2..8 vectors, long rows cut into K segments over the
warps of a CTA): per term, ws(k) = 1 (k <= 256) else min(8, ceil(k /
256)) segments of whole 16-column steps, each four interleaved k-ascending
chains of correctly rounded FMAs (chain j: columns 4j .. 4j + 3 of every
16-column step) summed as (c0 + c1) + (c2 + c3), segments left to right. Ragged row counts (not multiples
of the 8-row group), k not a multiple of the 16-column step, several segments,
the gathered second term (x2[idx2]), y0, several vectors with their own
strides. A column of a several-vector launch does not depend on how many
vectors share the launch."""
from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def chain(a, x):
    k = len(a)
    ws = 1 if k <= 256 else min(8, (k + 255) // 256)
    sl = ((-(-k // ws)) + 15) // 16 * 16
    total = None
    for s in range(ws):
        acc = [0.0, 0.0, 0.0, 0.0]
        for q in range(s * sl, min(k, (s + 1) * sl)):
            j = ((q - s * sl) % 16) // 4  # chain of the column within its 16-column step
            acc[j] = fma(a[q], x[q], acc[j])
        p = (acc[0] + acc[1]) + (acc[2] + acc[3])
        total = p if total is None else total + p
    return total


def lanes(a, x):
    s = [0.0] * 32
    for q in range(len(a)):
        s[q % 32] = fma(a[q], x[q], s[q % 32])
    for o in (16, 8, 4, 2, 1):
        s = [s[l] + s[l + o] if l + o < 32 else s[l] for l in range(32)]
    return s[0]


def make_jobs(rng, nv):
    buf = []
    idx = []

    def put(arr):
        off = sum(len(b) for b in buf)
        buf.append(np.ascontiguousarray(arr, dtype=np.float64).ravel())
        return off

    jobs = []
    shapes = [(1, 3, 0), (5, 16, 0), (8, 17, 9), (13, 50, 0), (37, 33, 21), (64, 130, 0), (70, 7, 40), (3, 0, 12),
              (9, 300, 0), (4, 700, 257), (2, 2100, 0)]
    for (m, k1, k2) in shapes:
        lda1 = k1 + int(rng.integers(0, 3))
        lda2 = k2 + int(rng.integers(0, 3))
        A1 = rng.standard_normal((m, max(lda1, 1)))
        A2 = rng.standard_normal((m, max(lda2, 1))) if k2 else None
        x1 = rng.standard_normal((nv, max(k1, 1)))
        nx2 = k2 + 11
        x2 = rng.standard_normal((nv, nx2)) if k2 else None
        y0 = rng.standard_normal((nv, m)) if m % 2 else None
        j = dict(m=m, k1=k1, k2=k2, A1=A1, A2=A2, x1=x1, x2=x2, y0=y0, a1=float(rng.choice([1.0, -1.0, 0.5])),
                 a2=float(rng.choice([1.0, -1.0])))
        j["A1o"] = put(A1)
        j["lda1"] = max(lda1, 1)
        j["x1o"] = put(x1)
        j["x1s"] = x1.shape[1]
        if k2:
            j["A2o"] = put(A2)
            j["lda2"] = max(lda2, 1)
            j["x2o"] = put(x2)
            j["x2s"] = nx2
            ii = rng.permutation(nx2)[:k2]
            j["ix"] = ii
            j["idxo"] = len(idx)
            idx.extend(ii.tolist())
        j["y0o"] = put(y0) if y0 is not None else -1
        j["yo"] = put(np.full((nv, m), np.nan))
        jobs.append(j)
    return jobs, np.concatenate(buf), np.array(idx, dtype=np.int64)


def reference(j, v, dot, fused):
    """y = y0; y += a1 s1; y += a2 s2, each update rounded twice or (contracted) once."""
    out = np.empty(j["m"])
    for i in range(j["m"]):
        y = j["y0"][v, i] if j["y0"] is not None else 0.0
        for a, A, k, xv in ((j["a1"], j["A1"], j["k1"], lambda: j["x1"][v, :j["k1"]]),
                            (j["a2"], j["A2"], j["k2"], lambda: j["x2"][v, j["ix"]] if j["k2"] else None)):
            if k:
                s = dot(A[i, :k], xv())
                y = fma(a, s, y) if fused else y + a * s
        out[i] = y
    return out


def run(jobs, buf, idx, nv):
    from paper_1410_2697_b200 import _lib
    desc = []
    ab = []
    for j in jobs:
        desc += [j["m"], j["k1"], j["k2"], j["yo"], j["y0o"], j["A1o"], j["lda1"], j["x1o"],
                 j.get("A2o", -1), j.get("lda2", 0), j.get("x2o", -1), j.get("idxo", -1),
                 j["m"], j["m"], j["x1s"], j.get("x2s", 0)]
        ab += [j["a1"], j["a2"]]
    desc = np.array(desc, dtype=np.int64)
    ab = np.array(ab, dtype=np.float64)
    out = buf.copy()
    ix = idx if len(idx) else np.zeros(1, dtype=np.int64)
    _lib.check(_lib.lib().mfh_test_gemv_batched(_lib.context().handle, len(jobs), _lib.ptr(desc), _lib.ptr(ab),
                                                _lib.ptr(out), out.size, _lib.ptr(ix), len(idx), nv))
    return out


@pytest.mark.parametrize("nv", [1, 2, 3, 8])
def test_gemv_bitwise_against_host_arithmetic(nv):
    rng = np.random.default_rng(7 + nv)
    jobs, buf, idx = make_jobs(rng, nv)
    out = run(jobs, buf, idx, nv)
    dot = lanes if nv == 1 else chain
    for j in jobs:
        got = out[j["yo"]:j["yo"] + nv * j["m"]].reshape(nv, j["m"])
        for v in range(nv):
            # the epilogue y + a * s may be contracted to one FMA: accept either
            # rounding of that step, nothing else
            ok = (got[v] == reference(j, v, dot, False)) | (got[v] == reference(j, v, dot, True))
            assert ok.all(), (nv, j["m"], j["k1"], j["k2"], v)


def test_gemv_columns_independent_of_batch_width():
    """Vector v of an 8-vector launch equals the 2-vector launch holding it
    (tensor-core path) bit for bit, and the one-vector launch (warp-per-row
    path) to rounding."""
    rng = np.random.default_rng(3)
    jobs, buf, idx = make_jobs(rng, 8)
    out8 = run(jobs, buf, idx, 8)
    for v in (0, 5, 6):
        for width in (2, 1):
            jv = []
            for j in jobs:
                q = dict(j)
                q["x1o"] = j["x1o"] + v * j["x1s"]
                if j["k2"]:
                    q["x2o"] = j["x2o"] + v * j["x2s"]
                if j["y0o"] >= 0:
                    q["y0o"] = j["y0o"] + v * j["m"]
                q["yo"] = j["yo"] + v * j["m"]
                jv.append(q)
            if width == 2 and v == 7:
                continue
            outw = run(jv, buf.copy(), idx, width)
            for j in jobs:
                a = out8[j["yo"] + v * j["m"]:j["yo"] + (v + 1) * j["m"]]
                b = outw[j["yo"] + v * j["m"]:j["yo"] + (v + 1) * j["m"]]
                if width == 2:
                    np.testing.assert_array_equal(a, b)
                else:
                    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12 * np.abs(a).max())
