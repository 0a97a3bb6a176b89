"""The CPU oracle (test infrastructure) pinned against the REFERENCE:
golden vectors produced by the reference's own rng.cpp/transforms.cpp
(tests/golden/make_golden.py), direct comparison with oracle/_ref when it is
present, and the reference's own known-answer tests restated
(test_basis.cpp, test_transforms.cpp, test_model.cpp, test_randls.cpp)."""
import ctypes as C
import math

import numpy as np
import pytest

from _models import const_one_model, legendre_model, one_sparse, random_points
from conftest import rel
from paper_1907_05884_b200.model import BasisSpec, Model

TAGS = {"val": 0x76616C69, "sub": 0x73756273, "sk": 0x736B6574}


# ------------------------------------------------------- golden vectors ---
def test_golden_rng(golden, O):
    for (s, t), want in zip(golden["mix_seed_in"], golden["mix_seed_out"]):
        assert O.mix_seed(int(s), int(t)) == int(want)
    i = 0
    while f"swr_{i}" in golden:
        seed, n, k = (int(v) for v in golden[f"swr_{i}_args"])
        assert np.array_equal(O.sample_without_replacement(seed, n, k), golden[f"swr_{i}"])
        i += 1
    assert i >= 6


def test_golden_plans(golden, O):
    i = 0
    while f"plan_{i}_rows" in golden:
        q_pad, s, seed = (int(v) for v in golden[f"plan_{i}_args"])
        signs, rows, scale = O.make_plan(q_pad, s, seed)
        assert np.array_equal(rows, golden[f"plan_{i}_rows"])
        assert np.array_equal(np.packbits(signs < 0), golden[f"plan_{i}_negbits"])
        assert set(np.unique(signs)) <= {-1.0, 1.0}
        assert scale == math.sqrt(q_pad / s)
        i += 1
    assert i == 3


@pytest.mark.parametrize("n", [1, 2, 8, 64, 1024, 4096])
def test_golden_transforms(golden, O, n):
    x, z = golden[f"x_{n}"], golden[f"z_{n}"]
    assert np.array_equal(O.dct2(x), golden[f"dct_{n}"])
    assert np.array_equal(O.wht(x), golden[f"wht_{n}"])
    for inv in (0, 1):
        assert np.array_equal(O.fft_pow2(z, bool(inv)), golden[f"fft{inv}_{n}"])
        assert np.array_equal(O.unitary_fft(z, bool(inv)), golden[f"ufft{inv}_{n}"])


def test_golden_next_pow2(golden, O):
    for a, b in zip(golden["next_pow2_in"], golden["next_pow2_out"]):
        assert O.next_pow2(int(a)) == int(b)


# ------------------------------------------- direct pins against _ref ---
def _ref_or_skip(O):
    R = O.ref()
    if R is None:
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return R


@pytest.mark.parametrize("n", [1 << 10, 1 << 18])
def test_ref_dct_wht_bitexact_large(O, n):
    R = _ref_or_skip(O)
    x = np.random.default_rng(n).normal(size=n)
    for fn, ref in ((O.dct2, R.ref_dct2), (O.wht, R.ref_wht)):
        y = x.copy()
        assert ref(y.ctypes.data_as(C.POINTER(C.c_double)), C.c_uint64(n)) == 0
        assert np.array_equal(fn(x), y)


def test_ref_plan_c1_bitexact(O):
    R = _ref_or_skip(O)
    q_pad, s = 1 << 18, 16384
    seed = O.mix_seed(0, TAGS["sk"])
    sg = np.zeros(q_pad)
    rows = np.zeros(s, dtype=np.uint64)
    R.ref_plan_stream(C.c_uint64(seed), C.c_uint64(q_pad), C.c_uint64(s),
                      sg.ctypes.data_as(C.POINTER(C.c_double)),
                      rows.ctypes.data_as(C.POINTER(C.c_uint64)))
    signs, rows2, _ = O.make_plan(190000, s, seed)
    assert np.array_equal(signs, sg) and np.array_equal(rows2, rows)


def test_ref_parallel_chunks_match(O):
    """parallel.cpp:38-39 chunking (n/(4T)) is what the restatement uses."""
    R = _ref_or_skip(O)
    n, t = 1000, 4
    b = np.zeros(n, dtype=np.uint64)
    R.ref_parallel_chunks(C.c_uint64(n), C.c_int(t), b.ctypes.data_as(C.POINTER(C.c_uint64)))
    chunk = max(1, n // (4 * t))
    assert np.array_equal(b, (np.arange(n) // chunk) * chunk)


# ------------------------------------------------ basis KATs (restated) ---
def _leg_closed(n, t):
    p = [1.0, t, 0.5 * (3 * t * t - 1), 0.5 * (5 * t ** 3 - 3 * t),
         0.125 * (35 * t ** 4 - 30 * t * t + 3), 0.125 * (63 * t ** 5 - 70 * t ** 3 + 15 * t)][n]
    return math.sqrt(2 * n + 1) * p


def test_legendre_kats(O):
    v = O.eval_basis(1, -1.0, 1.0, 0.0)            # test_basis.cpp:37-42
    assert v[0] == 1.0 and v[1] == 0.0
    v = O.eval_basis(2, -1.0, 1.0, 1.0)            # :44-50
    assert np.allclose(v, [1.0, math.sqrt(3), math.sqrt(5)], rtol=1e-15, atol=0)
    rng = np.random.default_rng(3)                 # :52-63
    for t in rng.uniform(-1, 1, 200):
        out = O.legendre_values(5, t)
        for n in range(6):
            assert abs(out[n] - _leg_closed(n, t)) <= 1e-12 * max(1.0, abs(_leg_closed(n, t)))


def test_domain_map_and_clamp(O):
    for t in (-1.0, -0.3, 0.0, 0.7, 1.0):          # :165-174
        x = 2.0 + (t + 1.0) * 2.0
        assert np.abs(O.eval_basis(4, -1, 1, t) - O.eval_basis(4, 2.0, 6.0, x)).max() <= 1e-12
    edge = O.eval_basis(3, 0.0, 1.0, 1.0)         # :176-183
    close = O.eval_basis(3, 0.0, 1.0, 1.0 + 1e-13)
    assert np.array_equal(edge, close)
    for bad in (1.5, -0.5):
        with pytest.raises(O.OracleError) as e:
            O.eval_basis(3, 0.0, 1.0, bad)
        assert e.value.kind == "Domain"


def test_invalid_specs(O):                          # :185-190
    for args in ((-1, -1.0, 1.0), (65, -1.0, 1.0), (2, 1.0, 1.0), (2, 2.0, 1.0)):
        with pytest.raises(O.OracleError) as e:
            O.eval_basis(args[0], args[1], args[2], 0.0)
        assert e.value.kind == "Parameter"


# ------------------------------------------- transform KATs (restated) ---
def _dct_direct(x):
    n = x.size
    k = np.arange(n)[:, None]
    m = np.arange(n)[None, :]
    c = np.where(np.arange(n) == 0, math.sqrt(1.0 / n), math.sqrt(2.0 / n))
    return c * (np.cos(np.pi * k * (2 * m + 1) / (2 * n)) @ x)


def _wht_direct(x):
    n = x.size
    i = np.arange(n)
    h = np.array([[(-1) ** bin(a & b).count("1") for b in i] for a in i], dtype=float)
    return h @ x / math.sqrt(n)


@pytest.mark.parametrize("n", [1, 2, 16, 128])
def test_transforms_vs_direct(O, n):                # test_transforms.cpp:92-158
    x = np.random.default_rng(n + 1).normal(size=n)
    for got, want in ((O.dct2(x), _dct_direct(x)), (O.wht(x), _wht_direct(x))):
        assert np.abs(got - want).max() <= 1e-10 * max(1.0, np.linalg.norm(want))
        assert abs(np.linalg.norm(got) - np.linalg.norm(x)) <= 1e-10 * np.linalg.norm(x)
    z = x + 1j * np.random.default_rng(n).normal(size=n)
    assert np.abs(O.fft_pow2(z) - np.fft.fft(z)).max() <= 1e-10 * max(1.0, np.linalg.norm(z))
    back = O.fft_pow2(O.fft_pow2(z), inverse=True)
    assert np.abs(back - z).max() <= 1e-12 * np.linalg.norm(z)
    assert abs(np.linalg.norm(O.unitary_fft(z)) - np.linalg.norm(z)) <= 1e-10 * np.linalg.norm(z)
    y = O.wht(O.wht(x))
    assert np.abs(y - x).max() <= 1e-12 * max(np.linalg.norm(x), 1e-300)


# ------------------------------------------------ model KATs (restated) ---
def test_const_model_is_one(O):                    # test_model.cpp:113-123
    m = const_one_model()
    for x in (-1.0, -0.25, 0.0, 0.8, 1.0):
        for y in (-1.0, 0.5):
            assert abs(O.evaluate(m, [x, y, -y]) - 1.0) <= 1e-14


def test_linearity_in_core(O):                     # :125-137
    m = legendre_model((2, 2), 5)
    m2 = m.with_core(3.5 * m.core)
    for x in (-0.9, 0.1, 0.77):
        assert abs(O.evaluate(m2, [x, -x]) - 3.5 * O.evaluate(m, [x, -x])) <= 1e-14 * max(
            1.0, abs(3.5 * O.evaluate(m, [x, -x])))


def test_batch_equals_scalar_and_threads(O):       # :178-199
    m = legendre_model((3, 3), 17)
    pts = random_points(200, 2, 23)
    O.set_max_threads(1)
    v1 = O.evaluate_batch(m, pts)
    O.set_max_threads(4)
    v4 = O.evaluate_batch(m, pts)
    O.set_max_threads(0)
    assert np.array_equal(v1, v4)
    for i in range(200):
        assert v1[i] == O.evaluate(m, pts[i])


def test_out_of_domain_and_arity(O):               # :201-210
    m = Model(np.array([2.0]), [[one_sparse(BasisSpec.legendre(0, 0.0, 1.0), 0, 1.0)]])
    assert abs(O.evaluate(m, [0.5]) - 2.0) < 1e-15
    with pytest.raises(O.OracleError) as e:
        O.evaluate(m, [1.75])
    assert e.value.kind == "Domain"
    with pytest.raises(O.OracleError) as e:
        O.evaluate(m, [0.5, 0.5])
    assert e.value.kind == "Parameter"


# ----------------------------------------------- randls KATs (restated) ---
def test_design_rows_ones_and_kronecker(O):        # test_randls.cpp:75-116
    m = Model(np.full((1, 1), 2.5), [[one_sparse(BasisSpec.legendre(0), 0, 1.0)]] * 2)
    w = O.build_design_rows(m, random_points(12, 2, 3))
    assert w.shape == (12, 1) and np.abs(w - 1.0).max() <= 1e-15
    m = legendre_model((3, 2, 4), 7)
    pts = random_points(20, 3, 11)
    w = O.build_design_rows(m, pts)
    for q in range(20):
        v = [O.mode_values(m, k, pts[q, k]) for k in range(3)]
        kr = np.einsum("k,j,i->kji", v[2], v[1], v[0]).ravel()  # mode-0 fastest
        assert np.allclose(w[q], kr, rtol=1e-12, atol=0)
    m = legendre_model((4, 3, 2), 13)
    pts = random_points(64, 3, 17)
    w = O.build_design_rows(m, pts)
    direct = O.evaluate_batch(m, pts)
    assert np.abs(w @ m.core.reshape(-1, order="F") - direct).max() <= 1e-10 * max(
        1.0, np.abs(direct).max())


@pytest.mark.parametrize("t", ["dct", "wht", "fft"])
def test_full_sampling_preserves_normal_equations(O, t):  # :118-141
    w = random_points(24, 6, 19)
    u = random_points(24, 1, 23)[:, 0]
    a, b, padded = O.sketch(w, u, seed=5, sample_rows=32, transform=t)
    assert padded == 32
    g1, g2 = a.T @ a, w.T @ w
    assert np.abs(g1 - g2).max() <= 1e-10 * max(1.0, np.abs(g2).max())
    assert np.abs(a.T @ b - w.T @ u).max() <= 1e-10 * max(1.0, np.abs(w.T @ u).max())


def test_sketch_determinism_and_rejection(O):      # :185-206
    w = random_points(200, 8, 47)
    u = random_points(200, 1, 53)[:, 0]
    s1 = O.sketch(w, u, seed=99, sample_rows=64)
    s2 = O.sketch(w, u, seed=99, sample_rows=64)
    s3 = O.sketch(w, u, seed=100, sample_rows=64)
    assert np.array_equal(s1[0], s2[0]) and np.array_equal(s1[1], s2[1])
    assert not np.array_equal(s1[0], s3[0])
    with pytest.raises(O.OracleError) as e:
        O.sketch(random_points(8, 2, 41), random_points(8, 1, 43)[:, 0], sample_rows=9)
    assert e.value.kind == "Parameter"


def test_mixing_isometry(O):                       # :170-183
    w = random_points(100, 4, 37)
    for t in ("dct", "wht", "fft"):
        mixed = O.mixed_matrix(w, seed=11, transform=t)
        assert np.allclose(np.linalg.norm(mixed, axis=0), np.linalg.norm(w, axis=0), rtol=1e-10)


def test_reestimate_recovers_exact_and_planted(O):  # :255-288
    m = legendre_model((3, 2, 2), 79)
    pts = random_points(2000, 3, 83)
    vals = O.evaluate_batch(m, pts)
    core, info = O.reestimate_core(m, pts, vals, seed=17)
    assert rel(core, m.core.reshape(-1, order="F")) <= 1e-8
    assert info["residual_after"] <= 1e-8 and not info["rank_deficient"]
    m = legendre_model((2, 3, 2), 89)
    planted = m.core + 0.5 * np.random.default_rng(97).normal(size=m.core.shape)
    ground = m.with_core(planted)
    pts = random_points(4000, 3, 101)
    core, _ = O.reestimate_core(m, pts, O.evaluate_batch(ground, pts), seed=23, sample_rows=48)
    assert rel(core, planted.reshape(-1, order="F")) <= 1e-6


def test_reestimate_rejections(O):                 # :313-322
    m = legendre_model((2, 2), 113)
    pts = random_points(500, 2, 127)
    with pytest.raises(O.OracleError) as e:
        O.reestimate_core(m, pts, O.evaluate_batch(m, pts), sample_rows=4)
    assert e.value.kind == "Parameter"
    with pytest.raises(O.OracleError):
        O.reestimate_core(m, pts[:10], O.evaluate_batch(m, pts[:10]), sample_rows=20)


# ------------------------------------------------ wavelet KATs (restated) ---
def test_wavelet_kats(O):
    v = O.eval_basis(0, -1.0, 1.0, -0.5, family=1, resolution=1)   # test_basis.cpp:65-72
    assert np.allclose(v, [1.0, -1.0], rtol=1e-14, atol=1e-14)
    for i in range(8):                                             # :74-90
        x = -1.0 + (2.0 * i + 1.0) / 8.0
        v = O.eval_basis(0, -1.0, 1.0, x, family=1, resolution=2)
        assert v.size == 4 and int(np.sum(np.abs(v) > 1e-12)) == 3


@pytest.mark.parametrize("s,p", [(1, 1), (3, 2), (4, 1), (0, 3)])
def test_wavelet_orthonormality(O, s, p):                          # :92-118
    n = (p + 1) << s
    cells = 1 << s
    nodes, weights = O.gauss_legendre(p + 2)
    gram = np.zeros((n, n))
    for c in range(cells):
        a, b = -1.0 + 2.0 * c / cells, -1.0 + 2.0 * (c + 1) / cells
        for xq, wq in zip(nodes, weights):
            x = 0.5 * (a + b) + 0.5 * (b - a) * xq
            v = O.eval_basis(p, -1.0, 1.0, x, family=1, resolution=s)
            gram += 0.5 * wq * (b - a) / 2.0 * np.outer(v, v)
    assert np.abs(gram - np.eye(n)).max() <= 1e-10


def test_wavelet_spaces_nest(O):                                   # :134-155
    p = 1
    for s in (1, 2, 3):
        q = 4 * ((p + 1) << s)
        pts = -1.0 + 2.0 * (np.arange(q) + 0.5) / q
        dc = np.array([O.eval_basis(p, -1, 1, x, family=1, resolution=s - 1) for x in pts])
        df = np.array([O.eval_basis(p, -1, 1, x, family=1, resolution=s) for x in pts])
        sol = np.linalg.lstsq(df, dc, rcond=None)[0]
        assert np.abs(df @ sol - dc).max() <= 1e-10


def test_haar_mother_is_step(O):
    c = O.mother_coords(0)                                         # basis.cpp:177-187 signs
    assert np.allclose(c[:, 0] * np.sqrt(2.0), [-1.0, 1.0], atol=1e-14)
