"""GPU parity for evaluation (fstk_gpu_evaluate_batch & co. through the C-ABI)
against the CPU oracle and the reference's own evaluation tests.

Tolerance (north_star): fp64 values within 1e-12 relative L2 of the oracle.
Mode values are bit-exact (same rounding sequence as basis.cpp:49-61 and the
sparse dot of model.cpp:86-88)."""
import numpy as np
import pytest

import paper_1907_05884_b200 as F
from _models import const_one_model, legendre_model, one_sparse, random_points
from conftest import rel
from paper_1907_05884_b200 import synth
from paper_1907_05884_b200.model import BasisSpec, Model

pytestmark = pytest.mark.gpu
TOL = 1e-12

SHAPES = {
    "C1": ((16, 16, 16), (20, 20, 20), 12),
    "C2": ((32, 32, 32), (48, 48, 48), 24),
    "C3": ((48, 48, 32), (64, 64, 64), 24),
    "C4": ((16, 16, 16, 8), (32, 32, 32, 16), 12),
    "d1": ((5,), (7,), 4),
    "d2": ((7, 9), (6, 6), 5),
    "ragged": ((5, 13, 3), (9, 17, 4), 6),
    "wide_r1": ((8, 80, 3), (10, 64, 5), 7),
    "d5": ((3, 2, 4, 2, 3), (4, 4, 4, 4, 4), 3),
    "d6": ((3, 2, 2, 2, 2, 2), (4, 3, 3, 3, 3, 3), 3),
    "d7": ((2, 2, 2, 2, 2, 2, 2), (3, 3, 3, 3, 3, 3, 3), 2),
    "d8_max_order": ((2, 2, 2, 2, 2, 2, 2, 2), (3, 3, 2, 2, 2, 2, 2, 2), 2),
    "p64_cap_degree": ((4, 3, 2), (64, 64, 64), 24),
    "jc48_shared_kernel": ((48, 8, 2), (48, 8, 8), 12),
    "jc40": ((40, 6, 3), (20, 20, 20), 8),
    "p48_param_kernel_jc8": ((8, 8, 8), (48, 48, 48), 12),
}


@pytest.mark.parametrize("name", list(SHAPES))
def test_eval_parity_shapes(O, name):
    ranks, deg, nnz = SHAPES[name]
    m = synth.random_model(ranks, deg, nnz, seed=1)
    pts = synth.uniform_points(20000 if len(ranks) < 5 else 3000, len(ranks), seed=2)
    got = m.evaluate_batch(pts)
    want = O.evaluate_batch(m, pts)
    assert rel(got, want) <= TOL


def test_eval_parity_fitted_c1(O):
    m = synth.fitted_model(64, (16, 16, 16), 20, 12)
    pts = synth.uniform_points(200_000, 3, seed=0)
    assert rel(m.evaluate_batch(pts), O.evaluate_batch(m, pts)) <= TOL


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_mode_values_bit_exact(O, mode):
    m = synth.random_model((32, 32, 32), (48, 48, 48), 24, seed=4)
    x = np.concatenate([np.random.default_rng(mode).random(500), [0.0, 1.0, 1.0 + 1e-13, -1e-13]])
    got = m.mode_values(mode, x)
    want = np.stack([O.mode_values(m, mode, xi) for xi in x])
    assert np.array_equal(got, want)


def test_batch_equals_scalar_bitexact():            # test_model.cpp:178-199
    m = legendre_model((3, 3), 17)
    pts = random_points(200, 2, 23)
    v = m.evaluate_batch(pts)
    for i in range(200):
        assert v[i] == m.evaluate(pts[i])


def test_position_independence_large():
    """A point's value does not depend on its position in the batch (chunk and
    tile boundaries): a full C2-sized evaluation equals evaluations of ragged
    sub-slices bit for bit, and two runs are identical."""
    m = synth.random_model((32, 32, 32), (48, 48, 48), 24, seed=1)
    n = 1 << 22
    pts = synth.uniform_points(n, 3, seed=9)
    full = m.evaluate_batch(pts)
    assert np.array_equal(full, m.evaluate_batch(pts))
    for lo, hi in ((0, 1), (1, 130), (12345, 12345 + 3 * 128 + 7), (n - 1000, n),
                   (2_000_001, 2_000_001 + (1 << 21) + 3)):
        assert np.array_equal(m.evaluate_batch(pts[lo:hi]), full[lo:hi])


def test_device_api_matches_host_api():
    import torch

    m = synth.random_model((16, 16, 16, 8), (32, 32, 32, 16), 12, seed=3)
    pts = synth.uniform_points(100_003, 4, seed=5)
    host = m.evaluate_batch(pts)
    dp = torch.from_numpy(np.ascontiguousarray(pts.T)).cuda()
    dev = m.evaluate_device(dp).cpu().numpy()
    assert np.array_equal(host, dev)


def test_const_model_and_linearity():               # test_model.cpp:113-137
    m = const_one_model()
    pts = np.array([[x, y, -y] for x in (-1.0, -0.25, 0.0, 0.8, 1.0) for y in (-1.0, 0.5)])
    assert np.abs(m.evaluate_batch(pts) - 1.0).max() <= 1e-14
    m = synth.random_model((8, 8, 8), (10, 10, 10), 5, seed=2)
    pts = synth.uniform_points(1000, 3, seed=3)
    a = m.evaluate_batch(pts)
    b = m.with_core(3.5 * m.core).evaluate_batch(pts)
    assert np.abs(b - 3.5 * a).max() <= 1e-14 * max(1.0, np.abs(3.5 * a).max())


def test_domain_errors_and_clamp():                 # basis.cpp:215-222, test_model.cpp:201-210
    m = Model(np.array([2.0]), [[one_sparse(BasisSpec.legendre(0, 0.0, 1.0), 0, 1.0)]])
    assert m.evaluate([0.5]) == 2.0
    with pytest.raises(ValueError) as e:
        m.evaluate([1.75])
    assert e.value.kind == "Domain"
    with pytest.raises(ValueError) as e:
        m.evaluate([0.5, 0.5])
    assert e.value.kind == "Parameter"
    m = synth.random_model((4, 4, 4), (6, 6, 6), 3, seed=1)
    pts = synth.uniform_points(300_000, 3, seed=1)
    pts[250_001, 1] = 1.0 + 1e-13      # inside the slack: clamped, accepted
    ok = m.evaluate_batch(pts)
    edge = pts.copy()
    edge[250_001, 1] = 1.0
    assert np.array_equal(ok, m.evaluate_batch(edge))
    bad = pts.copy()
    bad[270_000, 2] = 1.5
    bad[280_000, 0] = -0.5
    with pytest.raises(ValueError) as e:
        m.evaluate_batch(bad)
    assert e.value.kind == "Domain" and e.value.index == 270_000 and e.value.mode == 2
    nan = pts.copy()
    nan[5, 0] = np.nan
    with pytest.raises(ValueError) as e:
        m.evaluate_batch(nan)
    assert e.value.index == 5


def test_empty_and_single():
    m = synth.random_model((4, 4, 4), (6, 6, 6), 3, seed=1)
    assert m.evaluate_batch(np.zeros((0, 3))).shape == (0,)
    assert m.evaluate_batch(np.full((1, 3), 0.5)).shape == (1,)


def test_fstk_round_trip_evaluates_bit_identically(tmp_path):  # test_model.cpp:276-309
    m = synth.random_model((6, 5, 7), (12, 10, 9), 5, seed=8, lo=0.0, hi=2.0)
    p = tmp_path / "m.fstk"
    m.save(str(p))
    back = F.load_model(str(p))
    pts = synth.uniform_points(1000, 3, seed=31) * 2.0
    assert np.array_equal(m.evaluate_batch(pts), back.evaluate_batch(pts))


@pytest.mark.parametrize("wav", [((1, 0),), ((1, 2), (3, 1)), ((5, 3),), ((0, 4), (2, 2))])
def test_wavelet_and_mixed_models(O, wav):
    """Modes mixing Legendre and multiwavelet functions:
    evaluation within 1e-12 of the oracle, mode values bit-exact."""
    m = synth.mixed_wavelet_model((5, 4, 3), wavelets=wav, legendre_p=6, nnz=5, seed=len(wav))
    pts = synth.uniform_points(20_000, 3, seed=7)
    pts[0] = [0.0, 0.5, 1.0]           # interval boundaries
    pts[1] = [0.25, 0.75, 0.125]
    assert rel(m.evaluate_batch(pts), O.evaluate_batch(m, pts)) <= TOL
    for k in range(3):
        got = m.mode_values(k, pts[:300, k])
        want = np.stack([O.mode_values(m, k, x) for x in pts[:300, k]])
        assert np.array_equal(got, want)


def test_haar_model_values():
    """s=1, p=0 Haar: [1, step] (test_basis.cpp:65-72) through a 1-mode model."""
    spec = BasisSpec.wavelet(1, 0)
    m = Model(np.array([1.0, 1.0]), [[one_sparse(spec, 0, 1.0), one_sparse(spec, 1, 1.0)]])
    v = m.mode_values(0, np.array([-0.5, 0.5]))
    assert np.allclose(v, [[1.0, -1.0], [1.0, 1.0]], atol=1e-14)


def test_native_library_is_what_ran():
    before = F.launch_count()
    m = synth.random_model((8, 8, 8), (6, 6, 6), 3, seed=1)
    m.evaluate_batch(synth.uniform_points(1000, 3, 1))
    assert F.launch_count() >= before + 2


def test_domain_error_index_in_later_device_chunk():
    """The device API reports the global (not chunk-relative) lowest bad row."""
    import torch

    m = synth.random_model((4, 4, 4), (6, 6, 6), 3, seed=1)
    n = (1 << 21) * 2 + 1000
    pts = synth.uniform_points(n, 3, seed=2)
    pts[(1 << 21) + 777, 1] = 3.0
    dp = torch.from_numpy(np.ascontiguousarray(pts.T)).cuda()
    with pytest.raises(ValueError) as e:
        m.evaluate_device(dp)
    assert e.value.kind == "Domain" and e.value.index == (1 << 21) + 777 and e.value.mode == 1


def test_grid_reconstruct_and_slice(O):
    """Separable grid evaluation equals point-wise evaluation of
    every node (reconstruct --grid, slice) within the evaluation tolerance."""
    m = synth.random_model((6, 5, 4), (8, 7, 6), 4, seed=11)
    sizes = (17, 9, 5)
    g = m.reconstruct_grid(sizes)
    assert g.shape == sizes
    nodes = [np.linspace(0.0, 1.0, s) for s in sizes]
    X, Y, Z = np.meshgrid(*nodes, indexing="ij")
    pts = np.stack([X.ravel(order="F"), Y.ravel(order="F"), Z.ravel(order="F")], axis=1)
    want = O.evaluate_batch(m, pts)
    assert rel(g.reshape(-1, order="F"), want) <= TOL
    sl = m.slice(2, 0, {1: 0.3}, width=7, height=6)   # mode_x=2 (w), mode_y=0 (h)
    ys = np.linspace(0, 1, 6)
    xs = np.linspace(0, 1, 7)
    ref = np.array([[O.evaluate(m, [y, 0.3, x]) for x in xs] for y in ys])
    assert sl.shape == (6, 7) and rel(sl, ref) <= TOL
    w = synth.mixed_wavelet_model((4, 3, 2), seed=2)
    gw = w.evaluate_grid([np.linspace(0, 1, 9), [0.5, 0.25], np.linspace(0, 1, 4)])
    Xw, Yw, Zw = np.meshgrid(np.linspace(0, 1, 9), [0.5, 0.25], np.linspace(0, 1, 4), indexing="ij")
    pw = np.stack([Xw.ravel(order="F"), Yw.ravel(order="F"), Zw.ravel(order="F")], axis=1)
    assert rel(gw.reshape(-1, order="F"), O.evaluate_batch(w, pw)) <= TOL
    with pytest.raises(ValueError) as e:
        m.evaluate_grid([[0.5], [0.2, 1.7], [0.1]])
    assert e.value.kind == "Domain" and e.value.mode == 1 and e.value.index == 1


def test_grid_mode_products_large_tiles(O):
    """The DMMA mode-product chain (fstk_grid.cu) over several 64 x 64 tiles,
    ragged edges and ranks above one 32-wide staging chunk equals point-wise
    evaluation (GPU batch, itself 1e-12 from the oracle) within 1e-12."""
    m = synth.random_model((40, 36, 8), (12, 12, 12), 6, seed=12)
    sizes = (130, 70, 3)
    g = m.reconstruct_grid(sizes)
    nodes = [np.array([i / (s - 1) for i in range(s)]) for s in sizes]
    X, Y, Z = np.meshgrid(*nodes, indexing="ij")
    pts = np.stack([X.ravel(order="F"), Y.ravel(order="F"), Z.ravel(order="F")], axis=1)
    want = m.evaluate_batch(pts)
    assert rel(g.reshape(-1, order="F"), want) <= 1e-12
    sub = np.random.default_rng(3).choice(len(pts), 2000, replace=False)
    assert rel(g.reshape(-1, order="F")[sub], O.evaluate_batch(m, pts[sub])) <= 1e-12


def test_evaluate_fields_shared_points(O):
    # BASELINE C5 shape in small: 8 seeded fields, one shared point set,
    # points uploaded once; each column equals the per-model batch bit for bit.
    models = [synth.random_model((6, 5, 4), (10, 10, 10), 5, seed=40 + f) for f in range(8)]
    pts = synth.uniform_points(50_000, 3, seed=41)
    out = F.evaluate_fields(models, pts)
    assert out.shape == (50_000, 8)
    for f, m in enumerate(models):
        assert np.array_equal(out[:, f], m.evaluate_batch(pts))
        assert rel(out[:, f], O.evaluate_batch(m, pts)) <= 1e-12


def test_boundary_and_slack_points_evaluate(O):
    # basis.cpp:215-222: points exactly on lo/hi and within +-1e-12 span are
    # clamped and evaluate like the boundary; the GPU agrees with the oracle.
    m = synth.random_model((6, 5, 4), (12, 12, 12), 5, seed=70)
    eps = 1e-12 * 0.999
    edge = np.array([[0.0, 1.0, 0.5], [1.0, 0.0, 0.0], [-eps, 1.0 + eps, 0.25],
                     [1.0 + eps, -eps, 1.0], [0.5, 0.5, 0.5]])
    got = m.evaluate_batch(np.asfortranarray(edge))
    want = O.evaluate_batch(m, np.asfortranarray(edge))
    assert rel(got, want) <= 1e-12
    clamped = np.clip(edge, 0.0, 1.0)
    assert np.array_equal(got, m.evaluate_batch(np.asfortranarray(clamped)))


def test_refit_d2_and_d4_parity(O):
    for ranks in ((6, 5), (3, 3, 2, 2)):
        m = synth.random_model(ranks, [6] * len(ranks), 4, seed=71)
        q = 20_000
        pts = synth.uniform_points(q, len(ranks), 72)
        vals = O.evaluate_batch(m, pts) + 1e-2 * np.random.default_rng(73).normal(size=q)
        new, _ = F.reestimate_core(m, pts, vals, seed=5)
        core_o, _ = O.reestimate_core(m, pts, vals, seed=5)
        assert rel(new.core.reshape(-1, order="F"), core_o) <= 1e-9


def test_set_devices_splits_host_evaluation():
    # Two replicas on the one GPU of this box exercise the multi-device path:
    # slabs evaluated concurrently give the single-device bits, and a domain
    # error reports the lowest offending index across slabs.
    m = synth.random_model((10, 8, 6), (16, 16, 16), 6, seed=80)
    pts = synth.uniform_points(500_001, 3, seed=81)
    one = m.evaluate_batch(pts)
    try:
        F.set_devices([0, 0, 0])
        m2 = synth.random_model((10, 8, 6), (16, 16, 16), 6, seed=80)
        assert np.array_equal(m2.evaluate_batch(pts), one)
        bad = pts.copy(order="F")
        bad[400_000, 1] = 2.0   # in the last slab
        bad[200_000, 2] = -3.0  # in the middle slab: the lower index wins
        with pytest.raises(F.FstkValueError) as ei:
            m2.evaluate_batch(bad)
        assert ei.value.index == 200_000 and ei.value.mode == 2
        m3 = m2.with_core(m2.core * 2.0)
        assert np.allclose(m3.evaluate_batch(pts[:1000]), 2.0 * one[:1000], rtol=1e-14, atol=0)
        with pytest.raises(F.FstkValueError):
            F.set_devices([99])
    finally:
        F.set_devices([])


def test_pageable_staging_matches_pinned_and_reports_domain_index():
    # Host buffers that are not pinned are staged through the library's pinned
    # double buffer (several chunks here): bit-identical to the pinned path,
    # and a domain error in the third chunk keeps its global index.
    import torch

    m = synth.random_model((8, 6, 5), (12, 12, 12), 5, seed=90)
    n = 5_000_000
    pts = synth.uniform_points(n, 3, seed=91)
    got = m.evaluate_batch(pts)
    pin = torch.empty((3, n), dtype=torch.float64).pin_memory()
    pin.numpy()[:] = pts.T
    po = torch.empty(n, dtype=torch.float64).pin_memory()
    m.evaluate_batch_into(pin.numpy().T, po.numpy())
    assert np.array_equal(got, po.numpy())
    bad = pts.copy(order="F")
    bad[4_500_001, 0] = -0.5
    with pytest.raises(F.FstkValueError) as ei:
        m.evaluate_batch(bad)
    assert ei.value.index == 4_500_001 and ei.value.mode == 0


@pytest.mark.parametrize("fam,p,res", [(0, 0, 0), (0, 7, 0), (0, 48, 0), (0, 64, 0), (1, 2, 1),
                                       (1, 3, 3), (1, 0, 4)])
def test_eval_basis_bitexact(O, fam, p, res):
    # fstk.eval_basis (module.cpp:152-156) on the GPU, bit-exact against the
    # oracle restatement of basis.cpp:226-234, scalar and vector x.
    spec = BasisSpec.legendre(p, 0.0, 2.0) if fam == 0 else BasisSpec.wavelet(res, p, 0.0, 2.0)
    xs = np.concatenate([[0.0, 2.0, 1.0, 1e-13, 2.0 - 1e-13],
                         np.random.default_rng(p + res).uniform(0, 2, 50)])
    got = F.eval_basis(spec, xs)
    for i, x in enumerate(xs):
        want = O.eval_basis(p, 0.0, 2.0, x, family=fam, resolution=res)
        assert np.array_equal(got[i], want)
    assert np.array_equal(F.eval_basis(spec, 0.5), got[0] * 0 + F.eval_basis(spec, np.array([0.5]))[0])
    with pytest.raises(F.FstkValueError):
        F.eval_basis(spec, 2.5)
