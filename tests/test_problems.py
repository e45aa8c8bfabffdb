"""Input generators (host)."""
import numpy as np
import pytest

from paper_1410_2697_b200 import problems as PR


def test_poisson_small_matrices():  # reference tests/test_problems.py KATs
    A, b = PR.gen_poisson7(1, 1, 1)
    np.testing.assert_array_equal(A.toarray(), [[6.0]])
    np.testing.assert_array_equal(b, [1.0])
    A, _ = PR.gen_poisson7(2, 1, 1)
    np.testing.assert_array_equal(A.toarray(), [[6.0, -1.0], [-1.0, 6.0]])
    A, _ = PR.gen_poisson7(3, 3, 3)
    d = A.toarray()
    assert np.linalg.eigvalsh(d).min() > 0
    deg = (d != 0).sum(1) - 1
    np.testing.assert_array_equal(d.sum(1), 6.0 - deg)
    assert A.symmetric
    with pytest.raises(ValueError):
        PR.gen_poisson7(0, 1, 1)


def test_poisson_matches_reference_vertex_order(oracle):
    # vid = i + nx*(j + ny*k), couplings -1 in x, y, z
    A, _ = PR.gen_poisson7(3, 2, 2)
    d = A.toarray()
    assert d[0, 1] == -1 and d[0, 3] == -1 and d[0, 6] == -1 and d[0, 2] == 0


def test_config_sizes():
    A, _ = PR.gen_q1_2d(128)
    assert A.n_rows == 16384 and A.nnz == 145924
    A, _ = PR.gen_poisson7(48, 48, 48)
    assert A.n_rows == 110592 and A.nnz == 760320


def test_q1_stencil_and_spd():
    A, _ = PR.gen_q1_2d(5)
    d = A.toarray()
    assert np.allclose(np.diag(d), 8 / 3)
    assert np.linalg.eigvalsh(d).min() > 0
    assert np.allclose(d, d.T)


def test_hex_and_delaunay_spd():
    A, _ = PR.gen_hex_q1(5, seed=1)
    d = A.toarray()
    assert np.linalg.eigvalsh(d).min() > 0 and (d != 0).sum(1).max() == 27
    A, _ = PR.gen_p1_delaunay(15, seed=2)
    d = A.toarray()
    assert np.linalg.eigvalsh(d).min() > 0 and np.allclose(d, d.T)


def test_seeded_rhs():
    a = PR.seeded_rhs(10, 3, "normal")
    np.testing.assert_array_equal(a, np.random.default_rng(3).standard_normal(10))
    u = PR.seeded_rhs(10, 3, "uniform")
    assert np.all(np.abs(u) <= 1)
