"""The reference's rank decision on the GPU (randls.cpp:112-123):
ColPivHouseholderQR's rank with Eigen's threshold min(m,n) eps max|R_ii|,
the QR solution when full rank, the CompleteOrthogonalDecomposition
minimum-norm solution otherwise.  Checked against the oracle restatement
(oracle.solve_system_rank, LAPACK dgeqp3) at the solver level and through
reestimate_core on designs with near-duplicate mode functions.

Tolerances.  The flag and the rank must be identical.  Two different
backward-stable QRs (LAPACK's dgeqp3 in the oracle, the GPU's TSQR + pivoted
QR) return least-squares solutions that agree only to about kappa eps, kappa
the condition number of the kept part of R (max|R_ii| / min kept |R_ii|), and
fitted values A x formed from such solutions carry the same cancellation.  So
solutions are compared to max(1e-9, 100 kappa eps) and fitted values to
max(1e-9, 10 kappa eps); well-conditioned systems therefore still meet the
1e-9 core bar."""
import numpy as np
import pytest

import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import refit as FR

pytestmark = pytest.mark.gpu

EPS = np.finfo(np.float64).eps


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def _orth(m, n, seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).normal(size=(m, n)))
    return q


def _graded(m, n, cond, seed):
    """A = U diag(s) V^T with singular values log-spaced over [1/cond, 1]."""
    s = np.logspace(0, -np.log10(cond), n)
    return np.asfortranarray(_orth(m, n, seed) * s @ _orth(n, n, seed + 1).T)


def _oracle_diag(a):
    import scipy.linalg as sla

    r = sla.qr(a, mode="r", pivoting=True)[0]
    return np.abs(np.diag(r))


def _oracle_margin(a):
    """min|R_ii| / max|R_ii| of the oracle's pivoted QR over Eigen's
    threshold factor (cases are built at least 3x away from 1)."""
    d = _oracle_diag(a)
    return d.min() / d.max() / (min(a.shape) * EPS)


def _tols(a):
    """(solution, fitted-value) tolerances from the kept part's condition."""
    d = _oracle_diag(a)
    kept = d[d > min(a.shape) * EPS * d.max()] if d.max() > 0 else d[:0]
    kappa = kept.max() / kept.min() if kept.size else 1.0
    return max(1e-9, 100 * kappa * EPS), max(1e-9, 10 * kappa * EPS)


@pytest.mark.parametrize("cond", [1e2, 1e7, 1e11, 1e13, 1e18])
def test_solve_system_graded_matches_oracle(O, cond):
    m, n = 600, 48
    a = _graded(m, n, cond, seed=int(np.log10(cond)))
    b = np.random.default_rng(7).normal(size=m)
    marg = _oracle_margin(a)
    assert marg > 3 or marg < 1 / 3, "test case too close to Eigen's threshold"
    want, wdef, wrank = O.solve_system_rank(a, b)
    got, gdef, grank = FR.solve_system(a, b)
    assert gdef == wdef and grank == wrank
    tx, tf = _tols(a)
    assert _rel(got, want) <= tx
    # fitted values and the residual of the (truncated) LS solution agree
    fit = a @ want
    assert _rel(a @ got, fit) <= tf
    assert abs(np.linalg.norm(b - a @ got) - np.linalg.norm(b - fit)) <= tf * np.linalg.norm(fit)


def test_solve_system_exact_duplicates_min_norm(O):
    rng = np.random.default_rng(3)
    base = rng.normal(size=(400, 20))
    a = np.asfortranarray(np.hstack([base, base[:, [2, 5, 5]]]))  # three duplicates
    b = rng.normal(size=400)
    want, wdef, wrank = O.solve_system_rank(a, b)
    got, gdef, grank = FR.solve_system(a, b)
    assert wdef and gdef and grank == wrank == 20
    # exact duplicates: the COD solution is the pseudo-inverse solution
    pinv = np.linalg.lstsq(a, b, rcond=None)[0]
    assert _rel(got, want) <= 1e-10 and _rel(got, pinv) <= 1e-10


def test_solve_system_tiny_column_is_deficient(O):
    """Eigen's threshold is not scale-invariant: a column 1e-16 times smaller
    than the rest is numerically dependent for the reference."""
    rng = np.random.default_rng(4)
    a = np.asfortranarray(rng.normal(size=(300, 12)))
    a[:, 7] *= 1e-16
    b = rng.normal(size=300)
    want, wdef, wrank = O.solve_system_rank(a, b)
    got, gdef, grank = FR.solve_system(a, b)
    assert wdef and gdef and grank == wrank == 11
    assert _rel(got, want) <= 1e-10


def test_solve_system_zero_and_single_column(O):
    a = np.zeros((50, 4), order="F")
    b = np.ones(50)
    got, gdef, grank = FR.solve_system(a, b)
    assert gdef and grank == 0 and np.all(got == 0)
    a1 = np.asfortranarray(np.arange(1.0, 51.0)[:, None])
    got, gdef, grank = FR.solve_system(a1, b)
    want, wdef, _ = O.solve_system_rank(a1, b)
    assert not gdef and not wdef and _rel(got, want) <= 1e-14


def test_solve_system_many_row_blocks(O):
    """More rows than one TSQR block: the streamed factor equals one QR."""
    m, n = 300_000, 600
    rng = np.random.default_rng(9)
    a = np.asfortranarray(rng.normal(size=(m, n)))
    a[:, 10] = a[:, 3] + 1e-9 * a[:, 11]
    b = rng.normal(size=m)
    want, wdef, wrank = O.solve_system_rank(a, b)
    got, gdef, grank = FR.solve_system(a, b)
    assert gdef == wdef and grank == wrank
    assert _rel(a @ got, a @ want) <= _tols(a)[1]


# ---- through reestimate_core: near-duplicate mode functions ---------------
def _near_dup_model(delta, ranks=(4, 3, 3), p=6, seed=0):
    """Mode 0's functions 0 and 1 are L1 and L1 + delta L5: cond(A) ~ 4.7/delta."""
    from _models import one_sparse
    from paper_1907_05884_b200.model import BasisSpec, Model, ModeFunction

    spec = BasisSpec.legendre(p)
    modes = [[one_sparse(spec, j, 1.0) for j in range(r)] for r in ranks]
    modes[0][0] = ModeFunction(spec, [(1, 1.0)])
    modes[0][1] = ModeFunction(spec, [(1, 1.0), (5, delta)] if delta > 0 else [(1, 1.0)])
    core = np.random.default_rng(seed).normal(size=ranks)
    return Model(np.asfortranarray(core), modes)


@pytest.mark.parametrize("cond", [1e7, 1e9, 1e11, 1e13, 1e16, np.inf])
def test_refit_rank_decision_near_duplicates(O, cond):
    from _models import random_points

    delta = 0.0 if np.isinf(cond) else 4.7 / cond
    m = _near_dup_model(delta)
    pts = random_points(20_000, 3, 5)
    vals = O.evaluate_batch(m, pts) + 1e-3 * np.random.default_rng(2).normal(size=20_000)
    a, b, _, _, _ = O.refit_system(m, pts, vals, seed=3)
    marg = _oracle_margin(a)
    assert marg > 3 or marg < 1 / 3, "test case too close to Eigen's threshold"
    core_o, info_o = O.reestimate_core(m, pts, vals, seed=3)
    new, info = F.reestimate_core(m, pts, vals, seed=3)
    core_g = new.core.reshape(-1, order="F")
    assert info["rank_deficient"] == info_o["rank_deficient"]
    tx, tf = _tols(a)
    # the core, and the sketched design's fitted values (min-norm or full LS)
    assert _rel(core_g, core_o) <= tx
    assert _rel(a @ core_g, a @ core_o) <= tf
    assert abs(info["residual_after"] - info_o["residual_after"]) <= 2 * tf
    # cond >= 1e7 leaves the Cholesky refinement's rounding floor (cond eps)
    # above its 1e-11 stall bar, so these systems are all decided by the QR.
    if info_o["rank_deficient"]:
        assert info["qr_path"]


def test_refit_well_conditioned_certified(O):
    """The usual full-rank refit never takes the QR path: the certificate
    passes and the core matches the oracle to 1e-9."""
    from paper_1907_05884_b200 import synth

    m = synth.random_model((6, 5, 4), (8, 8, 8), 4, seed=21)
    pts = synth.uniform_points(30_000, 3, seed=22)
    vals = O.evaluate_batch(m, pts) + 1e-3 * np.random.default_rng(23).normal(size=30_000)
    new, info = F.reestimate_core(m, pts, vals, seed=5)
    core_o, info_o = O.reestimate_core(m, pts, vals, seed=5)
    assert not info["rank_deficient"] and not info_o["rank_deficient"]
    assert not info["qr_path"] and info["sigma_ratio"] > 100 * 120 * EPS
    assert _rel(new.core.reshape(-1, order="F"), core_o) <= 1e-9
