"""Seeded synthetic workloads for the BASELINE.json configurations.

The reference measures on DNS data that is not available, and
its CLI synth kinds differ from BASELINE's fields (§0-6), so the configs are
built here from seed: points, the analytic fields BASELINE.json describes,
and functional sparse Tucker models.  Models are either seeded random
(sparse Legendre expansions that are near-orthonormal, as fitted singular
functions are) or fitted by an upstream stand-in (grid sampling -> fixed-rank
HOSVD -> greedy sparse Legendre fit), which is NOT part of the hot path and
runs in numpy only to produce realistic cores/factors.
"""
from __future__ import annotations

import numpy as np

from .model import BasisSpec, Model, ModelMetadata, ModeFunction

CONFIGS = {
    # name: (dim, N, ranks, degrees, nnz, sample_rows_factor)
    "C1": dict(d=3, n=200_000, ranks=(16, 16, 16), degrees=(20, 20, 20), nnz=12, m_factor=4,
               grid=64),
    "C2": dict(d=3, n=256 ** 3, ranks=(32, 32, 32), degrees=(48, 48, 48), nnz=24, m_factor=8,
               grid=256),
    "C3": dict(d=3, n=1 << 27, ranks=(48, 48, 32), degrees=(64, 64, 64), nnz=24, m_factor=0,
               grid=0),
    "C4": dict(d=4, n=1 << 28, ranks=(16, 16, 16, 8), degrees=(32, 32, 32, 16), nnz=12,
               m_factor=16, grid=0),
    "C5": dict(d=3, n=1 << 26, ranks=(32, 32, 32), degrees=(48, 48, 48), nnz=24, m_factor=8,
               grid=0),
}


# ---------------------------------------------------------------- points ---
def uniform_points(n: int, d: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.random((n, d)))


def jittered_mesh(m: int, seed: int, jitter: float = 0.4) -> np.ndarray:
    """Cell-centred m^3 mesh with uniform jitter +-jitter cell (stays in [0,1])."""
    rng = np.random.default_rng(seed)
    g = (np.arange(m) + 0.5) / m
    x, y, z = np.meshgrid(g, g, g, indexing="ij")
    p = np.stack([x.ravel(order="F"), y.ravel(order="F"), z.ravel(order="F")], axis=1)
    p += rng.uniform(-jitter, jitter, size=p.shape) / m
    return np.asfortranarray(p)


def flame_surface_mixture(n: int, seed: int) -> np.ndarray:
    """C3: 50% uniform, 50% within +-0.03 of the front z = 0.5 + 0.05 sin sin."""
    rng = np.random.default_rng(seed)
    p = rng.random((n, 3))
    h = n // 2
    x, y = p[h:, 0], p[h:, 1]
    z = front(x, y) + rng.uniform(-0.03, 0.03, size=x.shape)
    p[h:, 2] = np.clip(z, 0.0, 1.0)
    return np.asfortranarray(p)


# ---------------------------------------------------------------- fields ---
def front(x, y):
    return 0.5 + 0.05 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y)


def flame_field(p: np.ndarray, seed: int = 0, n_gauss: int = 0, noise: float = 1e-2,
                gauss_width=(0.02, 0.1)) -> np.ndarray:
    """BASELINE C1/C2 field: tanh front + Gaussian bump(s) + N(0, noise^2).
    noise = 1e-2 reads "N(0,1e-4)" as variance 1e-4 (SURVEY §8d note a)."""
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    f = np.tanh((z - front(x, y)) / 0.02)
    f = f + 0.1 * np.exp(-((x - 0.3) ** 2 + (y - 0.6) ** 2 + (z - 0.4) ** 2) / 0.01)
    rng = np.random.default_rng(seed + 7919)
    for _ in range(n_gauss):
        c = rng.random(3)
        w = rng.uniform(*gauss_width)
        a = rng.normal(0.0, 0.2)
        f = f + a * np.exp(-((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2) / (w * w))
    if noise > 0:
        f = f + rng.normal(0.0, noise, size=f.shape)
    return f


# ---------------------------------------------------------------- models ---
def random_model(ranks, degrees, nnz, seed=0, lo=0.0, hi=1.0, core_decay=1.0) -> Model:
    """Seeded model: function j of mode k = L_{pi(j)} + 0.3 * (sparse Gaussian on
    nnz-1 other indices, decaying with degree), coefficients sorted by index."""
    rng = np.random.default_rng(seed)
    d = len(ranks)
    modes = []
    for k in range(d):
        p = degrees[k] if np.ndim(degrees) else degrees
        n = p + 1
        r = ranks[k]
        lead = rng.permutation(n)[:r] if r <= n else rng.integers(0, n, r)
        fns = []
        for j in range(r):
            m = min(nnz, n)
            others = [i for i in rng.permutation(n) if i != lead[j]][: m - 1]
            idx = sorted([int(lead[j])] + [int(i) for i in others])
            c = {}
            for i in idx:
                c[i] = 1.0 if i == lead[j] else 0.3 * rng.normal() / np.sqrt(max(m - 1, 1)) / (
                    1.0 + 0.05 * i)
            fns.append(ModeFunction(BasisSpec.legendre(p, lo, hi), [(i, c[i]) for i in idx]))
        modes.append(fns)
    core = rng.normal(size=tuple(ranks))
    if core_decay:
        for k in range(d):
            shp = [1] * d
            shp[k] = ranks[k]
            core = core / (1.0 + np.arange(ranks[k]).reshape(shp)) ** core_decay
    return Model(np.asfortranarray(core), modes, ModelMetadata(grid_sizes=[0] * d))


def mixed_wavelet_model(ranks, wavelets=((1, 2), (3, 1)), legendre_p=6, nnz=5, seed=0,
                        lo=0.0, hi=1.0) -> Model:
    """Seeded model whose modes mix Legendre and multiwavelet functions (the
    CLI always offers a wavelet candidate, pipeline.cpp:341-343): function j
    of mode k uses basis j % (len(wavelets)+1) (0 = Legendre p)."""
    rng = np.random.default_rng(seed)
    specs = [BasisSpec.legendre(legendre_p, lo, hi)] + [BasisSpec.wavelet(s_, p_, lo, hi)
                                                        for s_, p_ in wavelets]
    modes = []
    for k, r in enumerate(ranks):
        fns = []
        for j in range(r):
            b = specs[(j + k) % len(specs)]
            dim = b.dimension()
            m = min(nnz, dim)
            idx = sorted(int(i) for i in rng.choice(dim, size=m, replace=False))
            fns.append(ModeFunction(b, [(i, float(rng.normal())) for i in idx]))
        modes.append(fns)
    core = rng.normal(size=tuple(ranks))
    return Model(np.asfortranarray(core), modes, ModelMetadata(grid_sizes=[0] * len(ranks)))


def _legendre_matrix(p: int, t: np.ndarray) -> np.ndarray:
    out = np.zeros((t.size, p + 1))
    pm1, pm0 = np.ones_like(t), t.copy()
    out[:, 0] = 1.0
    if p >= 1:
        out[:, 1] = np.sqrt(3.0) * t
    for n in range(1, p):
        pn1 = ((2 * n + 1) * t * pm0 - n * pm1) / (n + 1)
        pm1, pm0 = pm0, pn1
        out[:, n + 1] = np.sqrt(2.0 * (n + 1) + 1.0) * pn1
    return out


def _omp(phi: np.ndarray, z: np.ndarray, max_nnz: int):
    """Greedy orthogonal matching pursuit (upstream stand-in for LARS+LOO)."""
    support = []
    r = z.copy()
    coef = np.zeros(0)
    for _ in range(min(max_nnz, phi.shape[1])):
        c = np.abs(phi.T @ r)
        c[support] = -1
        support.append(int(np.argmax(c)))
        coef, *_ = np.linalg.lstsq(phi[:, support], z, rcond=None)
        r = z - phi[:, support] @ coef
        if np.linalg.norm(r) <= 1e-12 * max(np.linalg.norm(z), 1e-300):
            break
    order = np.argsort(support)
    return [(support[i], float(coef[i])) for i in order], np.linalg.norm(r) / max(
        np.linalg.norm(z), 1e-300)


def fitted_model(grid: int, ranks, degree: int, max_nnz: int, seed: int = 0,
                 n_gauss: int = 0) -> Model:
    """Upstream stand-in (NOT the hot path): sample the noise-free field on a
    node-centred grid^3 over [0,1]^3, fixed-rank HOSVD, sparse Legendre fits.
    Runs with single-threaded BLAS: the greedy sparse fits pick different
    indices when the eigen/least-squares rounding changes with the thread
    count, and every launch (plain python, torchrun's OMP_NUM_THREADS=1) must
    build the same model from the same seed."""
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover - the image ships threadpoolctl
        return _fitted_model(grid, ranks, degree, max_nnz, seed, n_gauss)
    with threadpool_limits(1):
        return _fitted_model(grid, ranks, degree, max_nnz, seed, n_gauss)


def _fitted_model(grid: int, ranks, degree: int, max_nnz: int, seed: int,
                  n_gauss: int) -> Model:
    g = np.linspace(0.0, 1.0, grid)
    x, y, z = np.meshgrid(g, g, g, indexing="ij")
    pts = np.stack([x.ravel(order="F"), y.ravel(order="F"), z.ravel(order="F")], axis=1)
    t = flame_field(pts, seed=seed, n_gauss=n_gauss, noise=0.0).reshape(
        (grid, grid, grid), order="F")
    factors = []
    for k in range(3):
        unf = np.moveaxis(t, k, 0).reshape(grid, -1)
        w, v = np.linalg.eigh(unf @ unf.T)
        factors.append(v[:, ::-1][:, : ranks[k]])
    core = t
    for k in range(3):
        core = np.moveaxis(np.tensordot(factors[k].T, np.moveaxis(core, k, 0), axes=1), 0, k)
    tref = 2.0 * g - 1.0
    phi = _legendre_matrix(degree, tref)
    modes = []
    for k in range(3):
        fns = []
        for j in range(ranks[k]):
            coeffs, res = _omp(phi, factors[k][:, j], max_nnz)
            fns.append(ModeFunction(BasisSpec.legendre(degree, 0.0, 1.0), coeffs,
                                    residual_rel=float(res)))
        modes.append(fns)
    return Model(np.asfortranarray(core), modes,
                 ModelMetadata(grid_sizes=[grid] * 3, provenance='{"origin":"synth.fitted_model"}'))
