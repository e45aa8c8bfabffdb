"""The factorization's batched GEMM (run_gemm: 64x64 DMMA tiles with
register-prefetched k slabs, identity strips, deterministic split-K, cuBLAS
for large plain GEMMs) against a host reference that evaluates every output
as the k-ascending chain of correctly rounded FMAs (exact rational arithmetic,
then one rounding per step) and the kernel's epilogue alpha*acc (+ beta*C as
one FMA): bit for bit, at sizes that are not multiples of the tile, for the
aliased in-place TRSM job (C == B), disjoint blocks of one buffer and split-K.
The sharded-equals-single guarantee rests on this order."""
import ctypes as C
from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def ref_gemm(A, B, Cin, alpha, beta, split=0):
    """k-ascending FMA chain per output; with split-K, one chain per k chunk
    and the chunk partials summed in order (k_gemm_reduce)."""
    m, k = A.shape
    n = B.shape[1]
    out = np.empty((m, n))
    chunks = [(0, k)] if not split or k < 2 * split else [(c, min(k, c + split)) for c in range(0, k, split)]
    for i in range(m):
        for j in range(n):
            acc = None
            for (c0, c1) in chunks:
                part = 0.0
                for q in range(c0, c1):
                    part = fma(A[i, q], B[q, j], part)
                acc = part if acc is None else acc + part
            v = alpha * acc
            out[i, j] = v if beta == 0.0 else fma(beta, Cin[i, j], v)
    return out


def run(jobs, buf, split_k=0):
    from paper_1410_2697_b200 import _lib
    desc = np.array([j[:9] for j in jobs], dtype=np.int64).ravel()
    ab = np.array([j[9:] for j in jobs], dtype=np.float64).ravel()
    out = np.ascontiguousarray(buf.copy())
    _lib.check(_lib.lib().mfh_test_gemm_batched(_lib.context().handle, len(jobs), _lib.ptr(desc), _lib.ptr(ab),
                                                _lib.ptr(out), out.size, int(split_k)))
    return out


def view(buf, off, r, c, ld):
    return np.lib.stride_tricks.as_strided(buf[off:], shape=(r, c), strides=(8 * ld, 8)).copy()


@pytest.mark.parametrize("split_k", [0, 16])
def test_gemm_bitwise_against_fma_chain(split_k):
    rng = np.random.default_rng(1)
    shapes = [(1, 1, 1), (37, 45, 5), (64, 64, 16), (70, 33, 40), (5, 70, 67), (65, 1, 33)]
    buf_parts, jobs, meta = [], [], []
    off = 0
    for (m, n, k) in shapes:
        A = rng.standard_normal((m, k))
        B = rng.standard_normal((k, n))
        Cm = rng.standard_normal((m, n))
        alpha, beta = (1.0, 0.0) if (m + n) % 2 else (-1.0, 1.0)
        a0, b0, c0 = off, off + m * k, off + m * k + k * n
        buf_parts += [A.ravel(), B.ravel(), Cm.ravel()]
        off = c0 + m * n
        jobs.append((m, n, k, a0, b0, c0, k, n, n, alpha, beta))
        meta.append((A, B, Cm, alpha, beta, c0, m, n))
    buf = np.concatenate(buf_parts)
    out = run(jobs, buf, split_k)
    for (A, B, Cm, alpha, beta, c0, m, n) in meta:
        np.testing.assert_array_equal(view(out, c0, m, n, n), ref_gemm(A, B, Cm, alpha, beta, split_k))


def test_gemm_aliased_and_disjoint_blocks():
    """B <- T B in place (the TRSM job: C == B, m = k <= 64), and C, A, B as
    disjoint blocks of one row-major matrix (F_ff -= F_fp Gpf shape)."""
    rng = np.random.default_rng(2)
    w, ncol = 40, 57
    T = rng.standard_normal((w, w))
    B = rng.standard_normal((w, ncol))
    buf = np.concatenate([T.ravel(), B.ravel()])
    out = run([(w, ncol, w, 0, w * w, w * w, w, ncol, ncol, 1.0, 0.0)], buf)
    np.testing.assert_array_equal(view(out, w * w, w, ncol, ncol), ref_gemm(T, B, B, 1.0, 0.0))
    nh, npv = 90, 30  # F (nh x nh): F_ff(60x60) -= F_fp(60x30) @ G(30x60), G stored after F
    F = rng.standard_normal((nh, nh))
    G = rng.standard_normal((npv, nh - npv))
    buf = np.concatenate([F.ravel(), G.ravel()])
    job = (nh - npv, nh - npv, npv, npv * nh, nh * nh, npv * nh + npv, nh, nh - npv, nh, -1.0, 1.0)
    out = run([job], buf)
    Fo = out[:nh * nh].reshape(nh, nh)
    ref = ref_gemm(F[npv:, :npv], G, F[npv:, npv:], -1.0, 1.0)
    np.testing.assert_array_equal(Fo[npv:, npv:], ref)
    np.testing.assert_array_equal(Fo[:npv], F[:npv])  # nothing outside C is touched
    np.testing.assert_array_equal(Fo[npv:, :npv], F[npv:, :npv])


def test_gemm_identity_strip_and_library_route():
    """An identity operand (DenseBlock.as_factors' eye, leading dimension -1)
    is a scaled copy; a large plain GEMM goes to cuBLAS by default (rounding-level match)."""
    rng = np.random.default_rng(3)
    m, n = 33, 29
    B = rng.standard_normal((m, n))
    Cm = rng.standard_normal((m, n))
    buf = np.concatenate([B.ravel(), Cm.ravel()])
    out = run([(m, n, m, -1, 0, m * n, 0, n, n, -1.0, 1.0)], buf)
    np.testing.assert_array_equal(view(out, m * n, m, n, n), ref_gemm(np.eye(m), B, Cm, -1.0, 1.0))
    big = 600
    A = rng.standard_normal((big, big))
    Bb = rng.standard_normal((big, big))
    buf = np.concatenate([A.ravel(), Bb.ravel(), np.zeros(big * big)])
    out = run([(big, big, big, 0, big * big, 2 * big * big, big, big, big, 1.0, 0.0)], buf)
    got = view(out, 2 * big * big, big, big, big)
    assert np.max(np.abs(got - A @ Bb)) <= 1e-12 * big * np.max(np.abs(A @ Bb))


def test_large_gemm_kernel_bitwise_equals_tile_kernel():
    """k_gemm_big (128-wide tiles, 16-byte cp.async slabs) runs the same k-ascending DMMA chain
    and epilogue as k_gemm: the same bits on every large plain GEMM, for sizes ragged against
    both tilings, odd leading dimensions (8-byte copy path), an odd buffer offset, alpha / beta
    epilogues, and several jobs in one launch; and within rounding of cuBLAS."""
    rng = np.random.default_rng(11)
    shapes = [(600, 600, 600, 0, 1.0, 0.0), (513, 300, 901, 1, -1.0, 1.0), (1100, 129, 1003, 3, 0.5, -2.0),
              (257, 2050, 300, 0, 1.0, 1.0), (640, 64, 2048, 0, 1.0, 0.0), (1024, 1024, 130, 2, -1.0, 1.0)]
    parts, jobs, off = [], [], 1  # offset 1: operands 8-byte but not 16-byte aligned unless padded
    parts.append(np.zeros(1))
    for (m, n, k, pad, alpha, beta) in shapes:
        lda, ldb, ldc = k + pad, n + pad, n + pad
        if pad == 0 and off % 2:   # aligned jobs start on an even offset
            parts.append(np.zeros(1))
            off += 1
        ao, bo, co = off, off + m * lda, off + m * lda + k * ldb
        for sz in (m * lda, k * ldb, m * ldc):
            parts.append(rng.standard_normal(sz))
        off = co + m * ldc
        if (m * lda + k * ldb + m * ldc) % 2 and pad == 0:
            parts.append(np.zeros(1))
            off += 1
        jobs.append((m, n, k, ao, bo, co, lda, ldb, ldc, alpha, beta))
    buf = np.concatenate(parts)
    big = run(jobs, buf, -4)
    tiles = run(jobs, buf, -2)
    blas = run(jobs, buf, -3)
    np.testing.assert_array_equal(big, tiles)
    for (m, n, k, ao, bo, co, lda, ldb, ldc, alpha, beta) in jobs:
        A, B, Cm = view(buf, ao, m, k, lda), view(buf, bo, k, n, ldb), view(buf, co, m, n, ldc)
        ref = alpha * (A @ B) + beta * Cm
        got = view(big, co, m, n, ldc)
        assert np.max(np.abs(got - ref)) <= 1e-12 * k * np.max(np.abs(ref))
        assert np.max(np.abs(got - view(blas, co, m, n, ldc))) <= 1e-12 * k * np.max(np.abs(ref))
        if ldc > n:   # padding columns of C untouched
            np.testing.assert_array_equal(big[co + n:co + m * ldc:ldc][:m - 1], buf[co + n:co + m * ldc:ldc][:m - 1])
