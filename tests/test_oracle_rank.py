"""The oracle's restatement of solve_system (randls.cpp:112-123) on CPU:
Eigen's ColPivHouseholderQR rank rule and the COD minimum-norm fallback,
pinned by known answers (the reference's Eigen is absent, so these restate
its documented semantics: rank() counts |R_ii| > min(m,n) eps max|R_ii|;
CompleteOrthogonalDecomposition::solve returns the minimum-norm solution of
the rank-k truncation)."""
import numpy as np

EPS = np.finfo(np.float64).eps


def test_rank_rule_on_orthogonal_columns(O):
    # Orthogonal columns: the pivoted R is diag(column norms), sorted.
    m, n = 200, 5
    q, _ = np.linalg.qr(np.random.default_rng(0).normal(size=(m, n)))
    s = np.array([1e-3, 3.0, 0.4 * n * EPS * 3.0, 1.0, 0.5])
    a = q * s
    b = np.random.default_rng(1).normal(size=m)
    x, deficient, rank = O.solve_system_rank(a, b)
    assert deficient and rank == 4  # only 0.4 n eps max falls below the threshold
    # min-norm of the truncation: the dropped column gets coefficient 0
    assert abs(x[2]) <= 1e-12
    want = (q.T @ b) / s
    keep = [0, 1, 3, 4]
    assert np.allclose(x[keep], want[keep], rtol=1e-12, atol=0)


def test_cod_equals_pseudo_inverse_on_exact_deficiency(O):
    rng = np.random.default_rng(2)
    base = rng.normal(size=(100, 6))
    a = np.hstack([base, base[:, :2] + base[:, 2:4]])  # rank 6 of 8
    b = rng.normal(size=100)
    x, deficient, rank = O.solve_system_rank(a, b)
    assert deficient and rank == 6
    pinv = np.linalg.lstsq(a, b, rcond=None)[0]
    assert np.linalg.norm(x - pinv) <= 1e-12 * np.linalg.norm(pinv)


def test_full_rank_is_the_least_squares_solution(O):
    rng = np.random.default_rng(3)
    a = rng.normal(size=(80, 10))
    b = rng.normal(size=80)
    x, deficient, rank = O.solve_system_rank(a, b)
    assert not deficient and rank == 10
    assert np.linalg.norm(x - np.linalg.lstsq(a, b, rcond=None)[0]) <= 1e-13 * np.linalg.norm(x)


def test_zero_matrix_rank_zero(O):
    x, deficient, rank = O.solve_system_rank(np.zeros((10, 3)), np.ones(10))
    assert deficient and rank == 0 and np.all(x == 0)
