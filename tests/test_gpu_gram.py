"""The sliced int8 tensor-core Gram (fstk_gram.cu) through the C-ABI
(fstk_gpu_gram_device / the refit stages).

Bars: every entry within the rigorous digit-plane bound
    |G - A^T A|_ab <= 4 (ns + 3) 2^(-7 ns) rows max|A_a| max|A_b|
(+ the fp64 reference's own rounding); bit-exact when the entries need no
more bits than the planes hold; the refit core with the sliced Gram equal to
the native-Gram core to 1e-12 and to the oracle's QR core to the north-star
1e-9; systems the sliced Gram cannot precondition escalate (more planes, then the
native Gram) and land on the native answer; a Gram upgraded by the extra
plane sums equals the higher-precision Gram."""
import numpy as np
import pytest

import paper_1907_05884_b200 as F
from conftest import rel
from paper_1907_05884_b200 import synth

pytestmark = pytest.mark.gpu
CORE_TOL = 1e-9


def _torch():
    import torch

    return torch


def _check_bound(a, g, ns):
    torch = _torch()
    ref = a.t() @ a
    rows = a.shape[0]
    mx = a.abs().amax(dim=0)
    bound = 4 * (ns + 3) * 2.0 ** (-7 * ns) * rows * (mx[:, None] * mx[None, :])
    nrm = torch.linalg.norm(a, dim=0)
    bound = bound + 4 * rows * 2.0 ** -53 * (nrm[:, None] * nrm[None, :])
    bound = bound + 4 * rows * 2.0 ** -1074  # products in the subnormal range round absolutely
    low = torch.tril(torch.ones_like(ref, dtype=torch.bool))
    err = (g - ref).abs()
    assert bool((err[low] <= bound[low]).all()), float((err - bound)[low].max())
    assert bool((g[~low] == 0).all())  # upper triangle untouched
    return err, ref, low


@pytest.mark.parametrize("rows,n", [(1000, 300), (70_000, 257), (333, 4000), (500, 5000),
                                    (17, 263), (4099, 1024)])
@pytest.mark.parametrize("ns", [7, 5, 3, 2])
def test_gram_within_digit_plane_bound(rows, n, ns):
    # Levels 3 and 2 (8 and 7 moduli: 23- and 19-bit entries; 2 is the default)
    # sit inside the bounds of three and two 7-bit planes.
    torch = _torch()
    gen = torch.Generator(device="cuda").manual_seed(rows * 7 + n)
    a = torch.randn(rows, n, dtype=torch.float64, device="cuda", generator=gen)
    g = F.gram(a, slices=ns)
    err, ref, low = _check_bound(a, g, ns)
    if ns == 7:
        assert float(torch.linalg.norm(err[low]) / torch.linalg.norm(ref[low])) < 1e-13


def test_gram_native_matches_torch():
    torch = _torch()
    a = torch.randn(3000, 700, dtype=torch.float64, device="cuda")
    g = F.gram(a, slices=0)
    ref = a.t() @ a
    low = torch.tril(torch.ones_like(ref, dtype=torch.bool))
    assert float((g - ref).abs()[low].max() / ref.abs().max()) < 1e-13


def test_gram_wild_column_scales_and_zero_columns():
    torch = _torch()
    rng = np.random.default_rng(5)
    rows, n = 20_000, 600
    a = torch.randn(rows, n, dtype=torch.float64, device="cuda")
    scales = torch.tensor(2.0 ** rng.integers(-40, 41, n), dtype=torch.float64, device="cuda")
    a = a * scales[None, :]
    a[:, 7] = 0.0
    a[:, 300] = 0.0
    a[123, 55] = 1e9  # one outlier dominating its column
    for ns in (7, 6, 4, 3, 2):
        g = F.gram(a, slices=ns)
        _check_bound(a, g, ns)
        assert bool((g[7, :] == 0).all()) and bool((g[:, 300] == 0).all())


def test_gram_bitexact_when_entries_fit_the_planes():
    # Integers below 2^11 need only the first two digit planes (6 + 7 bits):
    # every C_t is exact, no dropped term is nonzero, and the fp64 fold of
    # integer sums < 2^53 is exact.
    torch = _torch()
    rng = np.random.default_rng(9)
    rows, n = 40_000, 320
    ai = rng.integers(-2047, 2048, size=(rows, n))
    ai[:, 0] = 2047  # pin every column max to the same exponent ...
    ai[:, 1] = 0
    ai[0, :] = 2047  # ... then the planes hold every entry exactly
    a = torch.tensor(ai, dtype=torch.float64, device="cuda")
    af = ai.astype(np.float64)
    exact = af.T @ af  # integers below 2^38: exact in the fp64 BLAS product
    g = F.gram(a, slices=7).cpu().numpy()
    low = np.tril(np.ones((n, n), dtype=bool))
    assert np.array_equal(g[low], exact[low])


def test_gram_rejects_bad_arguments():
    torch = _torch()
    a = torch.randn(10, 300, dtype=torch.float64, device="cuda")
    with pytest.raises(F.FstkValueError):
        F.gram(a, slices=1)
    with pytest.raises(F.FstkValueError):
        F.gram(a, slices=8)


def _problem(ranks, q, seed, degree=8, nnz=5):
    m = synth.random_model(ranks, [degree] * len(ranks), nnz, seed=seed)
    pts = synth.uniform_points(q, len(ranks), seed + 1)
    vals = synth.flame_field(pts, seed=seed + 2) if len(ranks) == 3 else np.sin(pts.sum(axis=1))
    return m, pts, vals


@pytest.mark.parametrize("t", ["dct", "wht", "fft", "none"])
def test_sliced_refit_matches_native_and_oracle(O, t):
    m, pts, vals = _problem((8, 8, 6), 60_000, 11)
    prev = F.gram_slices(7)
    try:
        new_s, info_s = F.reestimate_core(m, pts, vals, seed=5, transform=t)
        F.gram_slices(0)
        new_n, info_n = F.reestimate_core(m, pts, vals, seed=5, transform=t)
    finally:
        F.gram_slices(prev)
    assert info_s["gram_slices"] == 7 and info_n["gram_slices"] == 0
    assert info_s["gram_int8_ops"] > 0 and info_n["gram_int8_ops"] == 0
    cs, cn = new_s.core.reshape(-1, order="F"), new_n.core.reshape(-1, order="F")
    assert rel(cs, cn) <= 1e-12
    core_o, _ = O.reestimate_core(m, pts, vals, seed=5, transform=t)
    assert rel(cs, core_o) <= CORE_TOL
    assert not info_s["rank_deficient"]


def test_sliced_refit_sharded_matches_oracle(O):
    # Two row shards on one GPU with the all-reduces done by hand: the
    # dist.py algorithm (summed sliced Grams, refinement with summed
    # corrections) lands on the oracle's QR core.
    torch = _torch()
    m, pts, vals = _problem((8, 8, 6), 60_000, 13)
    R = 8 * 8 * 6
    prev = F.gram_slices(7)
    sessions = []
    try:
        sessions = [F.RefitSession(m, pts, vals, seed=3, shard=k, shards=2) for k in range(2)]
        gs = [torch.empty(R * R, dtype=torch.float64, device="cuda") for _ in range(2)]
        rs = [torch.empty(R, dtype=torch.float64, device="cuda") for _ in range(2)]
        for s, g, r in zip(sessions, gs, rs):
            s.normal_equations(g, r)
            assert s.info.gram_slices == 7
        gsum, rsum = gs[0] + gs[1], rs[0] + rs[1]
        xs = [torch.empty_like(rsum) for _ in range(2)]
        for s, x in zip(sessions, xs):
            assert s.factor(gsum, rsum, x)
        for _ in range(4):
            parts = [torch.empty_like(rsum) for _ in range(2)]
            for s, x, p in zip(sessions, xs, parts):
                s.correction(x, p)
            tot = parts[0] + parts[1]
            for s, x in zip(sessions, xs):
                s.apply(tot, x)
        assert torch.equal(xs[0], xs[1])
        core = sessions[0].finish(xs[0])
        core_o, _ = O.reestimate_core(m, pts, vals, seed=3)
        assert rel(core, core_o) <= CORE_TOL
    finally:
        for s in sessions:
            s.close()
        F.gram_slices(prev)


def _ill_conditioned_model(seed=21):
    """Mode functions 0 and 1 nearly collinear in every mode: the design
    columns then have cond ~1e6 or worse."""
    m = synth.random_model((8, 8, 6), (8, 8, 8), 9, seed=seed)  # R = 384: sliced path
    modes = [list(mk) for mk in m.modes]
    for k in range(3):
        base = modes[k][0]
        coeffs = [(i, c * (1.0 + 1e-6 * (j + 1))) for j, (i, c) in enumerate(base.coeffs)]
        modes[k][1] = F.ModeFunction(base.basis, coeffs)
    return F.Model(m.core, modes, m.metadata)


@pytest.mark.parametrize("t", ["dct", "none"])
def test_sliced_gram_escalates_when_it_cannot_precondition(O, t):
    m = _ill_conditioned_model()
    pts = synth.uniform_points(40_000, 3, 2)
    vals = synth.flame_field(pts, seed=4)
    prev = F.gram_slices(4)
    try:
        new_s, info_s = F.reestimate_core(m, pts, vals, seed=8, transform=t)
        F.gram_slices(0)
        new_n, info_n = F.reestimate_core(m, pts, vals, seed=8, transform=t)
    finally:
        F.gram_slices(prev)
    # 4 planes (28 bits) cannot precondition cond(A)^2 ~ 1e12: the solve
    # escalates (7 planes, then the native Gram) and lands on the native answer.
    assert info_s["gram_slices"] in (0, 7)
    assert info_s["rank_deficient"] == info_n["rank_deficient"]
    assert rel(new_s.core.reshape(-1, order="F"), new_n.core.reshape(-1, order="F")) <= 1e-9


def test_gram_levels_converge_to_the_native_gram():
    # normal_equations_level(5 / 7 / 0): the sliced Grams approach the native
    # one as the precision level rises; A^T b is always the fp64 DGEMV.
    torch = _torch()
    m, pts, vals = _problem((8, 8, 6), 60_000, 17)
    R = 384
    sess = F.RefitSession(m, pts, vals, seed=2)
    out = {}
    try:
        for lvl in (2, 3, 5, 7, 0):
            g = torch.empty(R * R, dtype=torch.float64, device="cuda")
            r = torch.empty(R, dtype=torch.float64, device="cuda")
            sess.normal_equations_level(lvl, g, r)
            assert sess.info.gram_slices == lvl
            out[lvl] = (g.view(R, R).t(), r)
        with pytest.raises(F.FstkValueError):
            sess.normal_equations_level(9, g, r)
    finally:
        sess.close()
    low = torch.tril(torch.ones(R, R, dtype=torch.bool, device="cuda"))
    GN = out[0][0]
    d = torch.sqrt(torch.diagonal(GN))
    sc = d[:, None] * d[None, :]
    e7 = float(((out[7][0] - GN).abs() / sc)[low].max())
    e5 = float(((out[5][0] - GN).abs() / sc)[low].max())
    e3 = float(((out[3][0] - GN).abs() / sc)[low].max())
    e2 = float(((out[2][0] - GN).abs() / sc)[low].max())
    assert e7 < 1e-13 and e5 < 1e-9 and e7 < e5 and e5 < e3 < 1e-5 and e3 < e2 < 1e-4
    assert torch.equal(out[5][1], out[0][1]) and torch.equal(out[7][1], out[0][1])


def test_default_five_planes_refit_matches_oracle(O):
    m, pts, vals = _problem((8, 8, 6), 60_000, 19)
    prev = F.gram_slices(5)
    try:
        new, info = F.reestimate_core(m, pts, vals, seed=4)
    finally:
        F.gram_slices(prev)
    assert info["gram_slices"] in (5, 7)
    core_o, _ = O.reestimate_core(m, pts, vals, seed=4)
    assert rel(new.core.reshape(-1, order="F"), core_o) <= CORE_TOL


def test_gram_slices_setting_roundtrip():
    prev = F.gram_slices()
    try:
        assert F.gram_slices(5) == prev
        assert F.gram_slices() == 5
        F.gram_slices(12)
        assert F.gram_slices() == 7  # clamped to 2..7
        F.gram_slices(1)
        assert F.gram_slices() == 2
        F.gram_slices(0)
        assert F.gram_slices() == 0
    finally:
        F.gram_slices(prev)


def test_gram_tiny_and_huge_column_scales_stay_finite():
    # Column maxima near the bottom of the double range (1e-305: the scale
    # 2^(k - e) alone would overflow) and large ones: every entry stays
    # within the bound, and no NaN/Inf appears where the true Gram is finite.
    torch = _torch()
    rows, n = 5000, 300
    a = torch.randn(rows, n, dtype=torch.float64, device="cuda")
    a[:, 3] *= 1e-305
    a[:, 4] *= 1e-160
    a[:, 5] *= 1e150
    a[:, 6] = 0.0
    for ns in (4, 7):
        g = F.gram(a, slices=ns)
        assert bool(torch.isfinite(g).all())
        _check_bound(a, g, ns)


@pytest.mark.parametrize("n,nb,slices", [(8192, 2048, 5), (3000, 512, 7), (4096, 1024, 4)])
def test_blocked_cholesky_with_int8_trailing_updates(n, nb, slices):
    # chol_crt: cuSOLVER potrf on the diagonal blocks, DTRSM panels, and the
    # trailing G22 -= L21 L21^T through the CRT int8 Gram.  Its backward error
    # ||L L^T - G|| / ||G|| is set by the plane accuracy of the updates
    # (2^-(7 slices - 1) per entry, relative to the row maxima).
    torch = _torch()
    gen = torch.Generator(device="cuda").manual_seed(n + slices)
    x = torch.randn(n + 500, n, dtype=torch.float64, device="cuda", generator=gen)
    x *= torch.exp(torch.randn(n, dtype=torch.float64, device="cuda", generator=gen))  # column scales
    g = x.t() @ x
    gn = float(torch.linalg.norm(g))
    l, info = F.cholesky(g, slices=slices, nb=nb)
    assert info == 0
    assert bool((l.triu(1) == 0).all())
    back = float(torch.linalg.norm(l @ l.t() - g)) / gn
    assert back < {4: 1e-7, 5: 1e-9, 7: 1e-13}[slices], back
    l0, info0 = F.cholesky(g, slices=0)
    assert info0 == 0 and float(torch.linalg.norm(l0 @ l0.t() - g)) / gn < 1e-14


def test_blocked_cholesky_reports_indefinite():
    torch = _torch()
    n = 3000
    g = torch.eye(n, dtype=torch.float64, device="cuda")
    g[2600, 2600] = -1.0  # the fifth 512-panel is not positive definite
    _, info = F.cholesky(g, slices=5, nb=512)
    assert info != 0
    _, info0 = F.cholesky(g, slices=0)
    assert info0 != 0


@pytest.mark.parametrize("rows,n", [(1000, 300), (70_000, 257), (333, 4000), (4099, 5000),
                                    (17, 263), (40_000, 2600), (128, 512)])
@pytest.mark.parametrize("ns", [4, 7])
def test_tcgen05_syrk_engine_equals_library_gemms(rows, n, ns):
    # The hand-written tcgen05 SYRK (fstk_syrk.cu: lower-triangle tiles,
    # residues reduced in the epilogue) and the cuBLASLt IMMA GEMMs feed the
    # same Garner fold with congruent values: the Grams are identical bit for
    # bit -- across several row segments (rows > 32768), column blocks
    # (n > 2048) and ragged edges (n, rows not multiples of 256 / 128).
    torch = _torch()
    gen = torch.Generator(device="cuda").manual_seed(rows + 31 * n + ns)
    a = torch.randn(rows, n, dtype=torch.float64, device="cuda", generator=gen)
    a[:, n // 3] *= 2.0 ** 30
    prev = F.gram_engine("cublaslt")
    try:
        g_lib = F.gram(a, slices=ns)
        F.gram_engine("tcgen05")
        g_tc = F.gram(a, slices=ns)
    finally:
        F.gram_engine(prev)
    assert F.gram_engine() == prev
    assert torch.equal(g_tc, g_lib)
    _check_bound(a, g_tc, ns)


def test_tcgen05_syrk_exact_integer_gram():
    # Integer columns below 2^13 fit the level-4 integers exactly: the Gram is
    # the exact integer A^T A, so the tensor-core path is checked against
    # integer arithmetic, not only against the library engine.
    torch = _torch()
    rng = np.random.default_rng(21)
    rows, n = 33_000, 700
    ai = rng.integers(-8191, 8192, size=(rows, n))
    ai[0, :] = 8191
    a = torch.tensor(ai, dtype=torch.float64, device="cuda")
    # |products| < 2^26 summed over 33,000 rows stay below 2^53: the fp64 BLAS
    # product is the exact integer Gram (and fast, unlike int64 numpy).
    af = ai.astype(np.float64)
    exact = af.T @ af
    prev = F.gram_engine("tcgen05")
    try:
        g = F.gram(a, slices=4).cpu().numpy()
    finally:
        F.gram_engine(prev)
    low = np.tril(np.ones((n, n), dtype=bool))
    assert np.array_equal(g[low], exact[low])


def test_gram_engine_setting():
    assert F.gram_engine() in ("tcgen05", "cublaslt")
    with pytest.raises(ValueError):
        F.gram_engine("wgmma")


_VARIANT_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r})
import paper_1907_05884_b200 as F
gen = torch.Generator(device="cuda").manual_seed(77)
a = torch.randn(41_000, 2600, dtype=torch.float64, device="cuda", generator=gen)
F.gram_engine("tcgen05")
g = F.gram(a, slices=4)
F.gram_engine("cublaslt")
h = F.gram(a, slices=4)
print("EQUAL" if torch.equal(g, h) else "DIFFER")
"""


@pytest.mark.parametrize("env", [{"FSTK_SYRK_MODE": "block"}, {"FSTK_SYRK_MODE": "fused"},
                                 {"FSTK_SYRK_CLUSTER": "4"},
                                 {"FSTK_SYRK_MODE": "block", "FSTK_SYRK_CLUSTER": "4"}])
def test_tcgen05_syrk_variants_bit_identical(env):
    # Every tcgen05 SYRK variant (environment, read once per process, hence a
    # subprocess): two segments, two column blocks, ragged edges -- the Gram
    # equals the library engine's bit for bit.
    import os
    import subprocess
    import sys

    from conftest import ROOT

    r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT.format(root=ROOT)],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "EQUAL"


def test_default_level_by_transform(O):
    # The process default is CRT level 2 (19-bit entries on 7 moduli) for a
    # mixed sketch oversampled at least 8x, and level 3 for thinner sketches
    # (the reference's default M = 2.5 R) and for the unmixed estimator, whose
    # systems are worse conditioned; all land on the oracle's core.
    m, pts, vals = _problem((8, 8, 6), 60_000, 23)
    R = 384
    assert F.gram_slices() == 2
    new_8, info_8 = F.reestimate_core(m, pts, vals, seed=5, sample_rows=8 * R)
    new_d, info_d = F.reestimate_core(m, pts, vals, seed=5)
    new_n, info_n = F.reestimate_core(m, pts, vals, seed=5, sample_rows=8 * R, transform="none")
    # benign system: no escalation
    assert info_8["gram_slices"] == 2 and info_d["gram_slices"] == 3 and info_n["gram_slices"] == 3
    for new, kw in ((new_8, dict(sample_rows=8 * R)), (new_d, {}),
                    (new_n, dict(sample_rows=8 * R, transform="none"))):
        core_o, _ = O.reestimate_core(m, pts, vals, seed=5, **kw)
        assert rel(new.core.reshape(-1, order="F"), core_o) <= CORE_TOL
