"""Host input generators for the BASELINE.json configurations.

``gen_poisson7`` restates the reference generator (problems.py:35-64, configs
2 and 5). The other generators are new (the reference has none for configs 1,
3, 4) and build the matrices SURVEY.md §8(d) specifies:

* ``gen_q1_2d``    — C1: bilinear Q1 Laplacian on an n x n interior grid
  (9-point stencil, centre 8/3, neighbours -1/3), Dirichlet eliminated;
* ``gen_hex_q1``   — C3: trilinear Q1 diffusion on n^3 interior nodes with a
  per-element log-normal coefficient from a seed;
* ``gen_p1_delaunay`` — C4: P1 Laplacian on a jittered lattice triangulated
  by scipy's Delaunay.

All return (SparseMatrix, rhs) with a reference-style all-ones rhs; the
benchmark draws its seeded rhs separately (``seeded_rhs``).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .sparse import SparseMatrix


def gen_poisson7(nx, ny, nz):
    """7-point Laplacian, diagonal 6, couplings -1 (problems.py:35-64)."""
    if min(nx, ny, nz) < 1:
        raise ValueError("grid dimensions must be at least 1")
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64).reshape(nz, ny, nx)  # vid = i + nx*(j + ny*k)
    rows = [idx.ravel()]
    cols = [idx.ravel()]
    vals = [np.full(n, 6.0)]
    for a, b in ((idx[:, :, :-1], idx[:, :, 1:]), (idx[:, :-1, :], idx[:, 1:, :]),
                 (idx[:-1, :, :], idx[1:, :, :])):
        a, b = a.ravel(), b.ravel()
        rows += [a, b]
        cols += [b, a]
        vals += [np.full(a.size, -1.0), np.full(a.size, -1.0)]
    A = SparseMatrix.from_triplets(n, n, np.concatenate(rows), np.concatenate(cols),
                                   np.concatenate(vals), symmetric=True)
    return A, np.ones(n)


def gen_q1_2d(nx, ny=None):
    """Q1 FE Laplacian on nx*ny interior nodes of a uniform grid (C1): centre 8/3,
    all 8 neighbours -1/3, Dirichlet boundary eliminated."""
    ny = nx if ny is None else ny
    n = nx * ny
    J, I = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    J, I = J.ravel(), I.ravel()
    vid = lambda j, i: i + nx * j
    rows, cols, vals = [vid(J, I)], [vid(J, I)], [np.full(n, 8.0 / 3.0)]
    for dj, di in ((0, 1), (1, 0), (1, 1), (1, -1)):
        ok = (J + dj < ny) & (I + di >= 0) & (I + di < nx)
        a = vid(J[ok], I[ok])
        b = vid(J[ok] + dj, I[ok] + di)
        rows += [a, b]
        cols += [b, a]
        vals += [np.full(a.size, -1.0 / 3.0)] * 2
    A = SparseMatrix.from_triplets(n, n, np.concatenate(rows), np.concatenate(cols),
                                   np.concatenate(vals), symmetric=True)
    return A, np.ones(n)


_Q1_HEX = None


def _hex_stiffness():
    """Unit-cube trilinear element Laplacian (2x2x2 Gauss), 8x8; scale h in 3D."""
    global _Q1_HEX
    if _Q1_HEX is None:
        corners = np.array([[i, j, k] for k in (0, 1) for j in (0, 1) for i in (0, 1)], float)
        s = 2.0 * corners - 1.0
        g = np.array([-1.0, 1.0]) / np.sqrt(3.0)
        K = np.zeros((8, 8))
        for gx in g:
            for gy in g:
                for gz in g:
                    dN = np.stack([s[:, 0] * (1 + s[:, 1] * gy) * (1 + s[:, 2] * gz),
                                   (1 + s[:, 0] * gx) * s[:, 1] * (1 + s[:, 2] * gz),
                                   (1 + s[:, 0] * gx) * (1 + s[:, 1] * gy) * s[:, 2]], axis=1) / 8.0
                    dNdx = dN * 2.0
                    K += dNdx @ dNdx.T * 0.125
        _Q1_HEX = K
    return _Q1_HEX


def gen_hex_q1(n, seed=0, sigma=1.0):
    """C3: trilinear Q1 diffusion, n^3 interior nodes ((n+1)^3 elements, h=1/(n+1)),
    per-element kappa = exp(N(0, sigma^2)) from ``seed``, Dirichlet on the boundary."""
    ne = n + 1
    h = 1.0 / ne
    Ke = _hex_stiffness() * h  # 3D Laplacian scales as h^(d-2)
    rng = np.random.default_rng(seed)
    kappa = np.exp(sigma * rng.standard_normal(ne ** 3))
    m = ne + 1  # nodes per direction incl. boundary
    ii, jj, kk = np.meshgrid(np.arange(ne), np.arange(ne), np.arange(ne), indexing="ij")
    ii, jj, kk = ii.ravel(order="F"), jj.ravel(order="F"), kk.ravel(order="F")
    # element ordering: i fastest
    order = np.lexsort((ii, jj, kk))
    ii, jj, kk = ii[order], jj[order], kk[order]
    nodes = np.stack([(ii + di) + m * ((jj + dj) + m * (kk + dk))
                      for dk in (0, 1) for dj in (0, 1) for di in (0, 1)], axis=1)
    interior = np.full(m ** 3, -1, dtype=np.int64)
    c = np.arange(m)
    inside = (c > 0) & (c < m - 1)
    mask = inside[None, None, :] & inside[None, :, None] & inside[:, None, None]  # [k, j, i]
    interior[np.flatnonzero(mask.ravel())] = np.arange(n ** 3)
    loc = interior[nodes]
    r = np.repeat(loc, 8, axis=1).ravel()
    cidx = np.tile(loc, (1, 8)).ravel()
    v = (kappa[:, None] * Ke.ravel()[None, :]).ravel()
    keep = (r >= 0) & (cidx >= 0)
    N = n ** 3
    K = sp.coo_matrix((v[keep], (r[keep], cidx[keep])), shape=(N, N)).tocsc()
    K.sum_duplicates()
    K = (K + K.T) * 0.5
    return SparseMatrix(K.tocsc(), symmetric=True), np.ones(N)


def gen_p1_delaunay(nside, seed=0, jitter=0.3):
    """C4: P1 Laplacian on an nside x nside lattice of [0,1]^2, interior points
    jittered U[-jitter*h, +jitter*h] from ``seed``, Delaunay triangulation,
    Dirichlet on the boundary nodes."""
    from scipy.spatial import Delaunay

    h = 1.0 / (nside - 1)
    g = np.linspace(0.0, 1.0, nside)
    X, Y = np.meshgrid(g, g, indexing="xy")
    pts = np.stack([X.ravel(), Y.ravel()], axis=1)
    bnd = (np.isclose(pts[:, 0], 0) | np.isclose(pts[:, 0], 1) | np.isclose(pts[:, 1], 0)
           | np.isclose(pts[:, 1], 1))
    rng = np.random.default_rng(seed)
    pts[~bnd] += rng.uniform(-jitter * h, jitter * h, size=(int((~bnd).sum()), 2))
    tri = Delaunay(pts).simplices
    P = pts[tri]  # (T, 3, 2)
    d1 = P[:, 1] - P[:, 0]
    d2 = P[:, 2] - P[:, 0]
    area = 0.5 * np.abs(d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0])
    # gradients of barycentric functions
    e = np.stack([P[:, 2] - P[:, 1], P[:, 0] - P[:, 2], P[:, 1] - P[:, 0]], axis=1)  # (T,3,2)
    grad = np.stack([-e[:, :, 1], e[:, :, 0]], axis=2) / (2 * area)[:, None, None]
    Ke = np.einsum("tad,tbd->tab", grad, grad) * area[:, None, None]
    ids = np.full(len(pts), -1, dtype=np.int64)
    ids[~bnd] = np.arange(int((~bnd).sum()))
    loc = ids[tri]
    r = np.repeat(loc, 3, axis=1).ravel()
    c = np.tile(loc, (1, 3)).ravel()
    v = Ke.ravel()
    keep = (r >= 0) & (c >= 0)
    N = int((~bnd).sum())
    K = sp.coo_matrix((v[keep], (r[keep], c[keep])), shape=(N, N)).tocsc()
    K.sum_duplicates()
    K = (K + K.T) * 0.5
    return SparseMatrix(K.tocsc(), symmetric=True), np.ones(N)


def seeded_rhs(n, seed=0, dist="normal"):
    """RHS i.i.d. N(0,1) or U[-1,1] from ``np.random.default_rng(seed)``."""
    rng = np.random.default_rng(seed)
    if dist == "normal":
        return rng.standard_normal(n)
    if dist == "uniform":
        return rng.uniform(-1.0, 1.0, n)
    raise ValueError(f"unknown rhs distribution '{dist}'")
