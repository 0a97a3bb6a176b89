"""GPU parity for the randomized-LS refit (fstk_gpu_reestimate_core & the
staged refit) against the CPU oracle.

Bars (north_star): sampled-point indices bit-exact; the sketched system A, b
bit-exact (the GPU replays the reference butterflies and twiddles); refit core
within 1e-9 relative L2 of the oracle's QR solution."""
import numpy as np
import pytest

import paper_1907_05884_b200 as F
from _models import legendre_model, random_points
from conftest import rel
from paper_1907_05884_b200 import synth

pytestmark = pytest.mark.gpu
CORE_TOL = 1e-9


def _data(O, model, q, seed, noise=0.01):
    pts = synth.uniform_points(q, model.order, seed)
    vals = O.evaluate_batch(model, pts) + noise * np.random.default_rng(seed).normal(size=q)
    return pts, vals


@pytest.mark.parametrize("t", ["dct", "wht", "fft"])
@pytest.mark.parametrize("q,ranks,wsub", [(20_000, (4, 3, 2), 1 << 20), (5000, (3, 3, 2, 2), 3000),
                                          (70_000, (6, 5, 4), 40_000)])
def test_sketch_rows_and_core_parity(O, t, q, ranks, wsub):
    m = synth.random_model(ranks, [6] * len(ranks), 4, seed=3)
    pts, vals = _data(O, m, q, 4)
    sess = F.RefitSession(m, pts, vals, seed=17, transform=t, working_subset=wsub)
    a, b = sess.sketched()
    ao, bo, rows_o, _, info_o = O.refit_system(m, pts, vals, seed=17, transform=t,
                                               working_subset=wsub)
    assert np.array_equal(sess.rows(), rows_o)
    assert np.array_equal(a, ao) and np.array_equal(b, bo)
    sess.close()
    new, info = F.reestimate_core(m, pts, vals, seed=17, transform=t, working_subset=wsub)
    core_o, info_o = O.reestimate_core(m, pts, vals, seed=17, transform=t, working_subset=wsub)
    assert rel(new.core.reshape(-1, order="F"), core_o) <= CORE_TOL
    for k in ("sample_rows", "working_rows", "held_out", "rank_deficient"):
        assert info[k] == info_o[k]
    assert abs(info["residual_after"] - info_o["residual_after"]) <= 1e-9 * max(
        1.0, info_o["residual_after"])


def test_c1_refit_parity(O):
    """BASELINE C1: N=200k, ranks 16^3 (R=4096), M = 4R = 16384, DCT."""
    m = synth.fitted_model(64, (16, 16, 16), 20, 12)
    pts = synth.uniform_points(200_000, 3, seed=0)
    vals = synth.flame_field(pts, seed=0, noise=1e-2)
    new, info = F.reestimate_core(m, pts, vals, seed=0, sample_rows=16384)
    core_o, info_o = O.reestimate_core(m, pts, vals, seed=0, sample_rows=16384)
    assert info["working_rows"] == 190_000 and info["padded_rows"] == 1 << 18
    assert rel(new.core.reshape(-1, order="F"), core_o) <= CORE_TOL
    assert np.array_equal(F.RefitSession(m, pts, vals, seed=0, sample_rows=16384).rows(),
                          info_o["rows"])


def test_public_sketch_and_mixed_bitexact(O):
    rng = np.random.default_rng(0)
    for t in ("dct", "wht", "fft"):
        for q in (1, 2, 24, 100, 3000, 70_000):
            w, u = rng.random((q, 6)), rng.random(q)
            s = min(40, q)
            a1, b1, p1 = F.sketch(w, u, seed=5, sample_rows=s, transform=t)
            a2, b2, p2 = O.sketch(w, u, seed=5, sample_rows=s, transform=t)
            assert p1 == p2 and np.array_equal(a1, a2) and np.array_equal(b1, b2)
        w = rng.random((100, 4))
        assert np.array_equal(F.mixed_matrix(w, seed=11, transform=t),
                              O.mixed_matrix(w, seed=11, transform=t))


@pytest.mark.parametrize("t", ["dct", "wht", "fft"])
def test_full_sampling_preserves_normal_equations(t):  # test_randls.cpp:118-141
    w = random_points(24, 6, 19)
    u = random_points(24, 1, 23)[:, 0]
    a, b, padded = F.sketch(w, u, seed=5, sample_rows=32, transform=t)
    assert padded == 32
    assert np.abs(a.T @ a - w.T @ w).max() <= 1e-10 * max(1.0, np.abs(w.T @ w).max())
    assert np.abs(a.T @ b - w.T @ u).max() <= 1e-10 * max(1.0, np.abs(w.T @ u).max())


def test_design_rows(O):                             # test_randls.cpp:88-116
    m = legendre_model((4, 3, 2), 13)
    pts = random_points(64, 3, 17)
    w = F.build_design_rows(m, pts)
    assert np.array_equal(w, O.build_design_rows(m, pts))
    v = m.evaluate_batch(pts)
    assert np.abs(w @ m.core.reshape(-1, order="F") - v).max() <= 1e-10 * max(1, np.abs(v).max())


def test_recovers_exact_and_planted_core(O):        # test_randls.cpp:255-288
    m = legendre_model((3, 2, 2), 79)
    pts = random_points(2000, 3, 83)
    new, info = F.reestimate_core(m, pts, O.evaluate_batch(m, pts), seed=17)
    assert rel(new.core, m.core) <= 1e-8 and info["residual_after"] <= 1e-8
    assert not info["rank_deficient"]
    m = legendre_model((2, 3, 2), 89)
    planted = m.core + 0.5 * np.random.default_rng(97).normal(size=m.core.shape)
    ground = m.with_core(planted)
    pts = random_points(4000, 3, 101)
    new, _ = F.reestimate_core(m, pts, O.evaluate_batch(ground, pts), seed=23, sample_rows=48)
    assert rel(new.core, planted) <= 1e-6


def test_biased_core_improves_and_holdout(O):       # test_randls.cpp:290-311
    ground = legendre_model((3, 3), 103)
    biased = ground.core + 0.2 * np.random.default_rng(107).normal(size=(3, 3)) * np.linalg.norm(
        ground.core) / 3.0
    m = ground.with_core(biased)
    pts = random_points(3000, 2, 109)
    new, info = F.reestimate_core(m, pts, O.evaluate_batch(ground, pts), seed=29)
    assert info["residual_after"] <= info["residual_before"]
    assert info["residual_after"] <= 1e-6 and info["held_out"]
    _, info = F.reestimate_core(m, pts, O.evaluate_batch(ground, pts), seed=29,
                                validation_fraction=0.0)
    assert not info["held_out"]


def test_rejections():                               # test_randls.cpp:185-191, 313-322
    m = legendre_model((2, 2), 113)
    pts = random_points(500, 2, 127)
    vals = np.sin(pts[:, 0])
    with pytest.raises(ValueError) as e:
        F.reestimate_core(m, pts, vals, sample_rows=4)
    assert e.value.kind == "Parameter"
    with pytest.raises(ValueError):
        F.reestimate_core(m, pts[:10], vals[:10], sample_rows=20)
    with pytest.raises(ValueError):
        F.sketch(random_points(8, 2, 41), random_points(8, 1, 43)[:, 0], sample_rows=9)
    bad = vals.copy()
    bad[3] = np.inf
    with pytest.raises(ValueError) as e:
        F.reestimate_core(m, pts, bad)
    assert e.value.kind == "Data"
    with pytest.raises(ValueError) as e:
        F.reestimate_core(m, pts[:, :1], vals)
    assert e.value.kind == "Shape"


def test_rank_deficient_flagged(O):
    """Duplicate mode functions make W rank deficient: the flag is raised (as
    the reference's COD fallback does) and the fit still reproduces the data."""
    from _models import one_sparse
    from paper_1907_05884_b200.model import BasisSpec, Model

    spec = BasisSpec.legendre(2)
    modes = [[one_sparse(spec, 0, 1.0), one_sparse(spec, 1, 1.0), one_sparse(spec, 1, 1.0)],
             [one_sparse(spec, 0, 1.0), one_sparse(spec, 2, 1.0)]]
    m = Model(np.arange(6.0).reshape(3, 2), modes)
    pts = random_points(2000, 2, 5)
    vals = O.evaluate_batch(m, pts)
    new, info = F.reestimate_core(m, pts, vals, seed=3)
    _, info_o = O.reestimate_core(m, pts, vals, seed=3)
    assert info["rank_deficient"] and info_o["rank_deficient"]
    assert info["residual_after"] <= 1e-8


def test_sharded_rows_sum_to_full_system(O):
    """Row shards (multi-GPU refit) partition the sketched rows; their partial
    normal equations sum to the full system (host-checked on one GPU)."""
    import torch

    m = synth.random_model((4, 3, 3), (5, 5, 5), 3, seed=2)
    pts, vals = _data(O, m, 30_000, 6)
    R = 36
    full = F.RefitSession(m, pts, vals, seed=4)
    gf = torch.empty(R * R, dtype=torch.float64, device="cuda")
    rf = torch.empty(R, dtype=torch.float64, device="cuda")
    full.normal_equations(gf, rf)
    g = torch.zeros(R * R, dtype=torch.float64, device="cuda")
    r = torch.zeros(R, dtype=torch.float64, device="cuda")
    for s in range(3):
        sess = F.RefitSession(m, pts, vals, seed=4, shard=s, shards=3)
        gs = torch.empty_like(g)
        rs = torch.empty_like(r)
        sess.normal_equations(gs, rs)
        g += gs
        r += rs
        sess.close()
    low = np.tril(np.ones((R, R), dtype=bool))
    G1 = gf.cpu().numpy().reshape(R, R, order="F")[low]
    G2 = g.cpu().numpy().reshape(R, R, order="F")[low]
    assert np.abs(G1 - G2).max() <= 1e-12 * np.abs(G1).max()
    core = full.solve(g, r)
    core_o, _ = O.reestimate_core(m, pts, vals, seed=4)
    assert rel(core, core_o) <= CORE_TOL


def test_validation_point_out_of_domain_is_domain_error(O):
    """A held-out point outside the domain fails the refit with Domain, as the
    reference's relative_residual -> evaluate_batch does (randls.cpp:350-356)."""
    m = synth.random_model((3, 3, 2), (5, 5, 5), 3, seed=3)
    pts, vals = _data(O, m, 20_000, 4)
    sess = F.RefitSession(m, pts, vals, seed=17)
    rows_val = None
    sess.close()
    # locate a validation row via the oracle's split and push it out of the domain
    _, _, _, val_index, _ = O.refit_system(m, pts, vals, seed=17)
    bad = pts.copy()
    bad[int(val_index[5]), 0] = 7.0
    with pytest.raises(ValueError) as e:
        F.reestimate_core(m, bad, vals, seed=17)
    assert e.value.kind == "Domain" and e.value.index == int(val_index[5])


@pytest.mark.parametrize("t", ["dct", "wht"])
def test_wavelet_model_refit_parity(O, t):
    m = synth.mixed_wavelet_model((4, 3, 3), wavelets=((2, 1),), legendre_p=5, nnz=4, seed=9)
    pts, vals = _data(O, m, 30_000, 5)
    sess = F.RefitSession(m, pts, vals, seed=3, transform=t)
    a, b = sess.sketched()
    ao, bo, rows_o, _, _ = O.refit_system(m, pts, vals, seed=3, transform=t)
    assert np.array_equal(a, ao) and np.array_equal(b, bo)
    sess.close()
    new, _ = F.reestimate_core(m, pts, vals, seed=3, transform=t)
    core_o, _ = O.reestimate_core(m, pts, vals, seed=3, transform=t)
    assert rel(new.core.reshape(-1, order="F"), core_o) <= CORE_TOL


# ------------------------------------------------------ diagnostics (8f-3) ---
def test_leverage_scores(O):                        # test_randls.cpp:208-230
    n = 12
    q, _ = np.linalg.qr(random_points(n, n, 59))
    assert np.abs(F.leverage_scores(q) - 1.0).max() <= 1e-10
    w = random_points(200, 10, 61)
    sc = F.leverage_scores(w)
    assert abs(sc.sum() - 10.0) <= 1e-8 * 10 and sc.min() >= 0.0
    assert np.abs(sc - O.leverage_scores(w)).max() <= 1e-10
    w = random_points(50, 3, 67) * 1e-6
    w[7] = [1e6, 0, 0]
    assert abs(F.leverage_scores(w)[7] - 1.0) <= 1e-6
    with pytest.raises(ValueError):
        F.leverage_scores(random_points(3, 5, 1))


def test_mixing_spreads_leverage():                 # test_randls.cpp:232-253
    q, r = 4096, 64
    w = random_points(q, r, 71) * 1e-3
    rng = np.random.default_rng(73)
    for _ in range(10):
        w[rng.integers(0, q)] = 100.0 * rng.normal(size=r)
    pre = F.leverage_scores(w)
    assert pre.max() / pre.mean() >= 50.0
    post = F.leverage_scores(F.mixed_matrix(w, seed=7))
    assert post.max() / post.mean() <= 5.0


def test_self_convergence(O):                        # test_randls.cpp:324-355
    m = legendre_model((2, 2), 131)
    pts = random_points(1000, 2, 137)
    vals = O.evaluate_batch(m, pts) + 0.01 * np.random.default_rng(139).normal(size=1000)
    curve = F.self_convergence(m, pts, vals, [64, 64, 64], seed=31)
    assert len(curve) == 2 and curve[0][1] == 0.0 and curve[1][1] == 0.0
    m = legendre_model((2, 2, 2), 149)
    pts = random_points(3000, 3, 151)
    vals = O.evaluate_batch(m, pts)
    curve = F.self_convergence(m, pts, vals, [16, 32, 64, 128], seed=37)
    assert len(curve) == 3 and all(np.isfinite(dl) and dl <= 1e-8 for _, dl in curve)
    noisy = vals + 0.001 * np.random.default_rng(5).normal(size=vals.size)
    got = F.self_convergence(m, pts, noisy, [16, 40, 128], seed=3)
    want = O.self_convergence(m, pts, noisy, [16, 40, 128], seed=3)
    for (s1, a), (s2, b) in zip(got, want):
        assert s1 == s2 and abs(a - b) <= 1e-8 * max(1.0, abs(b))
    with pytest.raises(ValueError):
        F.self_convergence(m, pts, vals, [64])
    with pytest.raises(ValueError):
        F.self_convergence(m, pts, vals, [64, 32])


# --------------------------------------- transform = none (north_star K5) ---
@pytest.mark.parametrize("q,ranks,wsub,s", [(20_000, (4, 3, 2), 1 << 20, 0), (9_000, (3, 3, 2, 2), 6000, 500),
                                            (50_000, (6, 5, 4), 30_000, 4000)])
def test_none_transform_parity(O, q, ranks, wsub, s):
    """Uniformly sampled design rows (no mixing), A generated block by block:
    sampled rows and A/b bit-exact against the oracle extension, core 1e-9."""
    m = synth.random_model(ranks, [6] * len(ranks), 4, seed=3)
    pts, vals = _data(O, m, q, 4)
    sess = F.RefitSession(m, pts, vals, seed=17, transform="none", working_subset=wsub,
                          sample_rows=s)
    a, b = sess.sketched()
    ao, bo, rows_o, _, _ = O.refit_system(m, pts, vals, seed=17, transform="none",
                                          working_subset=wsub, sample_rows=s)
    assert np.array_equal(sess.rows(), rows_o)
    assert np.array_equal(a, ao) and np.array_equal(b, bo)
    sess.close()
    new, info = F.reestimate_core(m, pts, vals, seed=17, transform="none", working_subset=wsub,
                                  sample_rows=s)
    core_o, info_o = O.reestimate_core(m, pts, vals, seed=17, transform="none",
                                       working_subset=wsub, sample_rows=s)
    assert rel(new.core.reshape(-1, order="F"), core_o) <= CORE_TOL
    assert info["padded_rows"] == info_o["padded_rows"]


def test_none_transform_recovers_planted_core(O):
    m = legendre_model((2, 3, 2), 89)
    planted = m.core + 0.5 * np.random.default_rng(97).normal(size=m.core.shape)
    pts = random_points(4000, 3, 101)
    new, _ = F.reestimate_core(m, pts, O.evaluate_batch(m.with_core(planted), pts), seed=23,
                               sample_rows=48, transform="none")
    assert rel(new.core, planted) <= 1e-10
    with pytest.raises(ValueError):   # S > Q_w
        F.reestimate_core(m, pts[:100], O.evaluate_batch(m, pts[:100]), sample_rows=99,
                          transform="none")


@pytest.mark.parametrize("t", ["dct", "fft", "wht"])
def test_three_pass_sketch_bitexact(O, t):
    # working_subset above 2^20 makes q_pad = 2^21: the sketch takes three
    # transform passes (a middle pass reads and writes the intermediate).
    m = synth.random_model((3, 2, 2), [5, 5, 5], 3, seed=31)
    q = (1 << 21) + 50_000  # q_w = q - 100,000 validation rows < 2^21
    pts, vals = _data(O, m, q, 32)
    sess = F.RefitSession(m, pts, vals, seed=6, transform=t, working_subset=0, sample_rows=64)
    assert sess.info_dict()["padded_rows"] == 1 << 21
    a, b = sess.sketched()
    ao, bo, rows_o, _, _ = O.refit_system(m, pts, vals, seed=6, transform=t, working_subset=0,
                                          sample_rows=64)
    assert np.array_equal(sess.rows(), rows_o)
    assert np.array_equal(a, ao) and np.array_equal(b, bo)
    sess.close()


@pytest.mark.parametrize("t,q,s", [("dct", 1_200_000, 4096), ("fft", 1_200_000, 4096),
                                   ("dct", 700_000, 600_000), ("fft", 700_000, 30)])
def test_two_pass_1m_sketch_bitexact(O, t, q, s):
    # q_pad = 2^20: both warp-level transform passes (the C2/C4/C5 shape),
    # with a full working subset (q = 1.2M) and with 383k zero-padded rows.
    m = synth.random_model((3, 2, 2), [6, 6, 6], 3, seed=41)
    pts, vals = _data(O, m, q, 42)
    sess = F.RefitSession(m, pts, vals, seed=8, transform=t, sample_rows=s)
    assert sess.info_dict()["padded_rows"] == 1 << 20
    a, b = sess.sketched()
    ao, bo, rows_o, _, _ = O.refit_system(m, pts, vals, seed=8, transform=t, sample_rows=s)
    assert np.array_equal(sess.rows(), rows_o)
    assert np.array_equal(a, ao) and np.array_equal(b, bo)
    sess.close()


@pytest.mark.parametrize("t,ranks", [("dct", (2, 2, 2, 2)), ("wht", (3, 2, 2))])
def test_two_pass_1m_order4_and_wht_bitexact(O, t, ranks):
    # q_pad = 2^20 for a 4-mode model (warp first pass with four tables) and
    # for the real WHT (shared-memory passes only).
    m = synth.random_model(ranks, [5] * len(ranks), 3, seed=43)
    pts, vals = _data(O, m, 1_150_000, 44)
    sess = F.RefitSession(m, pts, vals, seed=9, transform=t, sample_rows=2048)
    assert sess.info_dict()["padded_rows"] == 1 << 20
    a, b = sess.sketched()
    ao, bo, rows_o, _, _ = O.refit_system(m, pts, vals, seed=9, transform=t, sample_rows=2048)
    assert np.array_equal(sess.rows(), rows_o)
    assert np.array_equal(a, ao) and np.array_equal(b, bo)
    sess.close()


def test_cached_device_blocks_reused_bit_identically():
    # A sketched system >= 256 MB (S x R = 131,072 x 512 fp64) goes through
    # the library's large-block cache: the second refit reuses the first's
    # blocks and must return the same core bit for bit; trimming hands them back.
    from paper_1907_05884_b200 import _lib

    _lib.trim_device_cache(-1)
    m = synth.random_model((8, 8, 8), (8, 8, 8), 5, seed=51)
    pts = synth.uniform_points(400_000, 3, seed=52)
    vals = m.evaluate_batch(pts) + 1e-3 * np.random.default_rng(53).normal(size=400_000)
    prev = _lib.set_device_cache(2)  # persistent: blocks survive between sessions
    try:
        a, ia = F.reestimate_core(m, pts, vals, seed=54, sample_rows=131_072)
        b, ib = F.reestimate_core(m, pts, vals, seed=54, sample_rows=131_072)
        assert np.array_equal(a.core, b.core)
        assert ia["residual_after"] == ib["residual_after"]
        assert _lib.trim_device_cache(-1) >= 256 << 20
        assert _lib.trim_device_cache(-1) == 0
    finally:
        _lib.set_device_cache(prev)
    # Default policy (per session): reestimate_core returns holding no cached
    # blocks, and the result is the same bits as on reused blocks.
    _lib.set_device_cache(1)
    c, _ = F.reestimate_core(m, pts, vals, seed=54, sample_rows=131_072)
    assert np.array_equal(a.core, c.core)
    assert _lib.trim_device_cache(-1) == 0


def test_pair_last_pass_variant_bitexact():
    # The opt-in barrier-free last pass (pair_pass2_kernel, FSTK_SKETCH_WARP2=1:
    # read once per process) must reproduce the oracle's A and b bit for bit
    # like the default kernel: the q_pad = 2^20 sketch tests (DCT and FFT, full
    # and zero-padded working sets, 4-mode model) and a column-sharded sketch
    # re-run in a child process with the flag set.
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FSTK_SKETCH_WARP2="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q",
                        os.path.join(root, "tests", "test_gpu_refit.py"),
                        os.path.join(root, "tests", "test_gpu_columns.py"),
                        "-k", "two_pass_1m or column"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
