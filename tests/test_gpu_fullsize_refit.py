"""Noisy refits at BASELINE's full sizes against the oracle (C2, C4, one C5
field): the reference estimator's sketched system and its solution.

A full-size sketched A (68.7 GB at C2, 137 GB at C4) cannot be formed by the
CPU oracle, so each run is checked through properties that hold at any size:
  * the S sampled rows equal the oracle's plan (make_plan on mix_seed(seed,
    0x736b6574), randls.cpp:61-75) bit for bit;
  * 64 seeded columns of A, plus b, equal the oracle's per-column sketch
    (design_column + sign + DCT + sampling, randls.cpp:44-105) bit for bit;
  * the returned core is the least-squares solution of that bit-exact A:
    within 1e-9 relative of the QR solution of the same A (a second session
    re-sketches A bit for bit -- the first one's Gram and Cholesky factor are
    gone, so even C4's 137 GB A leaves room -- then streaming TSQR on the GPU
    and R x = Q^T b), with a normal-equation residual ||A^T (b - A x)|| at the
    QR solution's level;
  * the reference's rank decision: full rank, certified by the Cholesky
    route, no QR path needed.
C2 is the bench's own workload (bench.workload: the fitted model and the
jittered-mesh flame field); C4 and C5 use seeded models of their shapes with
BASELINE's fields plus noise."""
import numpy as np
import pytest

import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import _lib, synth
from paper_1907_05884_b200.dist import refine_distributed

pytestmark = pytest.mark.gpu


def _refit_parity(O, model, pts, vals, S, seed=0, ncols=64):
    import torch

    R = int(np.prod(model.ranks))
    dev = torch.device("cuda", torch.cuda.current_device())
    sess = F.RefitSession(model, pts, vals, seed=seed, sample_rows=S)
    try:
        cols = np.sort(np.random.default_rng(seed + 99).choice(R, ncols, replace=False))
        cols = np.append(cols, R)  # b
        a_o, rows_o = O.refit_column_set(model, pts, vals, cols, seed=seed, sample_rows=S)
        assert np.array_equal(sess.rows(), rows_o)
        a_g = sess.sketched_columns(cols)
        assert a_g.shape == a_o.shape == (S, ncols + 1)
        assert np.array_equal(a_g, a_o)

        gram = _lib.device_tensor(R * R, dev)
        rhs = torch.empty(R, dtype=torch.float64, device=dev)
        sess.normal_equations(gram, rhs)
        x = refine_distributed(sess, gram, rhs)
        del gram, rhs
        core = sess.finish(x)
        info = sess.info_dict()
        assert not info["rank_deficient"] and not info["qr_path"]
        assert np.isfinite(core).all()
        s = torch.empty_like(x)
        sess.correction(x, s)
    finally:
        sess.close()
    torch.cuda.empty_cache()
    # The QR solution of the same (bit-exact, re-sketched) A.
    n1 = R + 1
    sess = F.RefitSession(model, pts, vals, seed=seed, sample_rows=S)
    try:
        raug = _lib.device_tensor(n1 * n1, dev)
        sess.local_qr(raug)
        rq = raug.view(n1, n1).t()  # column-major storage -> [row, col]
        x_qr = torch.linalg.solve_triangular(rq[:R, :R].contiguous(), rq[:R, R:].contiguous(),
                                             upper=True)[:, 0]
        del raug, rq
        torch.cuda.empty_cache()
        rel = float(torch.linalg.norm(x - x_qr) / torch.linalg.norm(x_qr))
        assert rel <= 1e-9, f"core vs QR solution of the same A: {rel:.3e}"
        s_qr = torch.empty_like(x)
        sess.correction(x_qr, s_qr)
        assert float(torch.linalg.norm(s)) <= 10 * float(torch.linalg.norm(s_qr))
    finally:
        sess.close()
    return core, info, rel


def test_c2_fullsize_noisy_refit_parity(O):
    import bench

    model, pts, vals, c = bench.workload("C2", 0, 0)
    R = int(np.prod(model.ranks))
    _, info, _ = _refit_parity(O, model, pts, vals, c["m_factor"] * R, seed=0)
    assert info["sample_rows"] == 262_144 and info["padded_rows"] == 1 << 20


def test_c4_fullsize_noisy_refit_parity(O):
    c = synth.CONFIGS["C4"]
    model = synth.random_model(c["ranks"], c["degrees"], c["nnz"], seed=4)
    rng = np.random.default_rng(41)
    n = 1 << 22
    pts = rng.random((n, 4))
    pts[:, 3] = rng.integers(0, 64, n) / 63.0
    x, y, z, t = pts.T
    vals = np.tanh((z - 0.3 - 0.4 * t - 0.05 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y)) / 0.02)
    vals = vals + 1e-2 * rng.normal(size=n)
    R = int(np.prod(model.ranks))
    _, info, _ = _refit_parity(O, model, np.asfortranarray(pts), vals, c["m_factor"] * R, seed=4)
    assert info["sample_rows"] == 524_288


def test_c5_field_fullsize_noisy_refit_parity(O):
    c = synth.CONFIGS["C5"]
    model = synth.random_model(c["ranks"], c["degrees"], c["nnz"], seed=5)
    pts = synth.uniform_points(1 << 22, 3, seed=51)
    vals = synth.flame_field(pts, seed=52, n_gauss=8)
    R = int(np.prod(model.ranks))
    _, info, _ = _refit_parity(O, model, pts, vals, c["m_factor"] * R, seed=5)
    assert info["sample_rows"] == 262_144
