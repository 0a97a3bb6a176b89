"""Multi-device refit behind the C-ABI (fstk_multi.cu): after
set_devices(n > 1) a model carries replicas and fstk_gpu_reestimate_core runs
the column-sharded sketch, the all-to-all, per-device partial normal
equations, one reduce of the packed triangles and the sharded refinement in
one process.  On this single-GPU pool the replicas share device 0 and the
peer-copy transport moves the data; the core must equal the single-device
core (same least-squares solution) and the oracle's."""
import numpy as np
import pytest

import paper_1907_05884_b200 as F
from conftest import rel
from paper_1907_05884_b200 import synth

pytestmark = pytest.mark.gpu


def _refit(ranks, degs, nnz, mseed, q, devices, **kw):
    try:
        F.set_devices(devices)
        m = synth.random_model(ranks, degs, nnz, seed=mseed)
        pts = synth.uniform_points(q, len(ranks), seed=mseed + 1)
        vals = m.evaluate_batch(pts) + 1e-3 * np.random.default_rng(mseed + 2).normal(size=q)
        new, info = F.reestimate_core(m, pts, vals, **kw)
    finally:
        F.set_devices([])
    return m, pts, vals, new, info


@pytest.mark.parametrize("transform,G", [("dct", 2), ("wht", 3), ("fft", 2), ("none", 2), ("dct", 4)])
def test_multi_device_refit_matches_single_and_oracle(O, transform, G):
    m, pts, vals, multi, info = _refit((6, 5, 4), (8, 8, 8), 4, 50, 30_000, [0] * G, seed=3,
                                       transform=transform)
    assert info["devices"] == G and info["transport"] == "p2p"
    one, info1 = F.reestimate_core(m, pts, vals, seed=3, transform=transform)
    a = multi.core.reshape(-1, order="F")
    b = one.core.reshape(-1, order="F")
    assert rel(a, b) <= 1e-12
    core_o, info_o = O.reestimate_core(m, pts, vals, seed=3, transform=transform)
    assert rel(a, core_o) <= 1e-9
    assert info["rank_deficient"] == info_o["rank_deficient"] is False
    assert abs(info["residual_after"] - info1["residual_after"]) <= 1e-12 * info1["residual_after"]


def test_multi_device_refit_int8_gram_path(O):
    # R >= 256: the sliced int8 Gram per device (tcgen05 SYRK), packed and
    # reduced; same core as one device to 1e-12, oracle to 1e-9.
    m, pts, vals, multi, info = _refit((8, 8, 6), (8, 8, 8), 5, 60, 40_000, [0, 0], seed=9)
    assert info["gram_slices"] > 0 and info["devices"] == 2
    one, _ = F.reestimate_core(m, pts, vals, seed=9)
    assert rel(multi.core.reshape(-1, order="F"), one.core.reshape(-1, order="F")) <= 1e-12
    core_o, _ = O.reestimate_core(m, pts, vals, seed=9)
    assert rel(multi.core.reshape(-1, order="F"), core_o) <= 1e-9


def test_multi_device_rank_deficient_takes_the_qr_path(O):
    # Duplicate mode functions: the sharded TSQR factors are stacked on the
    # solver device, pivoted QR decides rank as Eigen would, COD min-norm.
    base = synth.random_model((4, 3, 3), (6, 6, 6), 3, seed=70)
    modes = [list(mf) for mf in base.modes]
    modes[0][1] = modes[0][0]
    m = F.Model(base.core, modes)
    pts = synth.uniform_points(20_000, 3, seed=71)
    vals = O.evaluate_batch(m, pts) + 1e-3 * np.random.default_rng(72).normal(size=20_000)
    try:
        F.set_devices([0, 0])
        m2 = F.Model(base.core, modes)
        new, info = F.reestimate_core(m2, pts, vals, seed=4)
    finally:
        F.set_devices([])
    core_o, info_o = O.reestimate_core(m, pts, vals, seed=4)
    assert info["rank_deficient"] and info_o["rank_deficient"] and info["qr_path"]
    assert rel(new.core.reshape(-1, order="F"), core_o) <= 1e-9
