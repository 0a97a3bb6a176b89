"""The hot-path parts of the reference's own Python smoke test
(proj/python/tests/test_smoke.py), run against this package under the same
names -- the drop-in claim checked the way a reference user would.  The
upstream-only tests there (sthosvd, assemble, interpolate, synth fields) are
out of scope; where they built a model, a seeded model stands in."""
import os
import tempfile

import numpy as np
import pytest

import paper_1907_05884_b200 as fstk
from paper_1907_05884_b200 import synth

pytestmark = pytest.mark.gpu


def test_basis_eval():  # test_smoke.py:27-33, verbatim
    leg = fstk.BasisSpec.legendre(2)
    v = fstk.eval_basis(leg, 1.0)
    assert np.allclose(v, [1.0, np.sqrt(3.0), np.sqrt(5.0)], atol=1e-12)
    haar = fstk.BasisSpec.wavelet(1, 0)
    w = fstk.eval_basis(haar, -0.5)
    assert np.allclose(w, [1.0, -1.0], atol=1e-12)


def test_evaluate_save_load():  # test_smoke.py:36-56 without assemble()
    model = synth.mixed_wavelet_model((3, 2), wavelets=((3, 1),), legendre_p=10, seed=4)
    pts = np.array([[0.25, 0.5], [0.75, 0.125]])
    vals = model.evaluate_batch(pts)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "model.fstk")
        model.save(path)
        again = fstk.load_model(path)
        assert np.array_equal(again.evaluate_batch(pts), vals)
        assert again.ranks == model.ranks
    assert model.storage()["coefficients"] > 0
    assert model.compression_ratio(33 ** 2) > 1.0


def test_reestimate_core_refines():  # test_smoke.py:59-73 without sthosvd/assemble
    rng = np.random.default_rng(3)
    model = synth.random_model((4, 4), (8, 8), 5, seed=2)
    pts = rng.uniform(0.0, 1.0, size=(4000, 2))
    vals = np.exp(-pts[:, 0]) * (1.0 + pts[:, 1])
    new_model, info = fstk.reestimate_core(model, pts, vals, seed=1)
    assert info["sample_rows"] > np.prod(model.ranks)
    assert info["residual_after"] <= max(info["residual_before"], 1e-3)
    for key in ("residual_before", "residual_after", "sample_rows", "working_rows",
                "rank_deficient", "held_out"):  # module.cpp:282-287
        assert key in info
