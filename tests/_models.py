"""Model/point builders restating the reference test fixtures
(proj/tests/test_randls.cpp:35-67, test_model.cpp:64-70)."""
import numpy as np

from paper_1907_05884_b200.model import BasisSpec, Model, ModelMetadata, ModeFunction


def one_sparse(spec, index, value):
    return ModeFunction(spec, [(int(index), float(value))])


def legendre_model(ranks, seed):
    """test_randls.cpp:45-58: mode-k functions are the first r_k normalised
    Legendre polynomials on [-1, 1]; core ~ N(0, 1)."""
    rng = np.random.default_rng(seed)
    core = rng.normal(size=tuple(ranks))
    modes = []
    for r in ranks:
        spec = BasisSpec.legendre(r - 1)
        modes.append([one_sparse(spec, j, 1.0) for j in range(r)])
    return Model(np.asfortranarray(core), modes, ModelMetadata())


def random_points(q, d, seed, lo=-1.0, hi=1.0):
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.uniform(lo, hi, size=(q, d)))


def const_one_model():
    """test_model.cpp:113-123."""
    spec = BasisSpec.legendre(0)
    return Model(np.ones((1, 1, 1)), [[one_sparse(spec, 0, 1.0)] for _ in range(3)])
