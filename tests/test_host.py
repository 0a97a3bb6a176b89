"""Host-side logic that needs no GPU: FSTK container I/O (model.cpp:280-426),
model validation (model.cpp:22-53, basis.cpp:30-47), error classes
(module.cpp:112-125), synthetic workloads and the flop accounting."""
import os
import struct

import numpy as np
import pytest

import paper_1907_05884_b200 as F
from _models import legendre_model, one_sparse
from paper_1907_05884_b200 import synth
from paper_1907_05884_b200.model import BasisSpec, Model, ModeFunction


def test_fstk_round_trip_bit_exact(tmp_path):
    m = synth.random_model((4, 3, 5), (7, 6, 9), 4, seed=11)
    m.metadata.provenance = '{"origin":"unit-test"}'
    m.metadata.epsilon = 1e-9
    p = tmp_path / "m.fstk"
    m.save(str(p))
    b = F.load_model(str(p))
    assert b.ranks == m.ranks and np.array_equal(b.core, m.core)
    assert b.metadata.provenance == m.metadata.provenance and b.metadata.epsilon == 1e-9
    for k in range(3):
        for f1, f2 in zip(m.modes[k], b.modes[k]):
            assert f1.basis == f2.basis and f1.coeffs == f2.coeffs
    # the payload layout of format.md:56-69
    raw = p.read_bytes()
    assert raw[:4] == b"FSTK" and struct.unpack_from("<I", raw, 4)[0] == 1
    hlen = struct.unpack_from("<Q", raw, 8)[0]
    core = np.frombuffer(raw, "<f8", 60, 16 + hlen)
    assert np.array_equal(core, m.core.reshape(-1, order="F"))


def test_fstk_rejects_corrupt(tmp_path):           # test_model.cpp:311-330
    p = tmp_path / "bad.fstk"
    p.write_bytes(b"JUNKJUNKJUNKJUNK")
    with pytest.raises(OSError):
        F.load_model(str(p))
    m = Model(np.ones((1, 1)), [[one_sparse(BasisSpec.legendre(1), 0, 1.0)],
                                [one_sparse(BasisSpec.legendre(1), 1, 2.0)]])
    m.save(str(p))
    raw = p.read_bytes()
    p.write_bytes(raw[:-5])
    with pytest.raises(F.FstkIOError) as e:
        F.load_model(str(p))
    assert e.value.kind == "Decode"
    p.write_bytes(raw + b"x")
    with pytest.raises(F.FstkIOError):
        F.load_model(str(p))
    with pytest.raises(F.FstkIOError) as e:
        F.load_model(str(tmp_path / "missing.fstk"))
    assert e.value.kind == "Io"


def test_model_validation():
    spec = BasisSpec.legendre(2)
    with pytest.raises(ValueError):                  # rank mismatch
        Model(np.ones((2, 1)), [[one_sparse(spec, 0, 1.0)], [one_sparse(spec, 0, 1.0)]])
    with pytest.raises(ValueError):                  # index outside dimension
        Model(np.ones(1), [[one_sparse(spec, 3, 1.0)]])
    with pytest.raises(ValueError):                  # inconsistent domains
        Model(np.ones(2), [[one_sparse(spec, 0, 1.0),
                            one_sparse(BasisSpec.legendre(2, 0.0, 1.0), 0, 1.0)]])
    for bad in (lambda: BasisSpec.legendre(-1), lambda: BasisSpec.legendre(65),
                lambda: BasisSpec.legendre(2, 1.0, 1.0), lambda: BasisSpec.wavelet(-1, 0)):
        with pytest.raises(ValueError):
            bad()
    m = legendre_model((2, 3), 1)
    with pytest.raises(ValueError):
        m.with_core(np.ones((3, 2)))
    assert m.domain(1) == (-1.0, 1.0)


def test_storage_and_ratio():                       # test_model.cpp:212-274
    spec = BasisSpec.legendre(2)
    m = Model(np.ones((2, 2)), [[ModeFunction(spec, [(0, 1.0), (1, 2.0), (2, 3.0)])] * 2] * 2)
    s = m.storage()
    assert s["coefficients"] == 4 + 12 and s["index_bytes"] == 48
    assert m.compression_ratio(s["total_bytes"] // 8) == pytest.approx(1.0, rel=1e-15)


def test_error_classes():
    e = F.FstkValueError("Domain", "x", mode=1, index=5, value=2.0)
    assert isinstance(e, ValueError) and e.kind == "Domain" and e.index == 5
    assert isinstance(F.FstkIOError("Io", "y"), OSError)


def test_synth_workloads_in_domain():
    p = synth.jittered_mesh(16, 3)
    assert p.shape == (4096, 3) and p.min() > 0 and p.max() < 1
    q = synth.flame_surface_mixture(1000, 1)
    assert q.min() >= 0 and q.max() <= 1
    f = synth.flame_field(p, n_gauss=8)
    assert np.all(np.isfinite(f))
    m = synth.fitted_model(32, (4, 4, 4), 10, 6)
    assert m.ranks == [4, 4, 4]
    assert all(len(fn.coeffs) <= 6 for mm in m.modes for fn in mm)


def test_flop_accounting_matches_survey():
    import bench

    m = synth.random_model((32, 32, 32), (48, 48, 48), 24, seed=0)
    fc, fm = bench.flops_per_point(m)
    assert fc == 67648 and fm == 5472
    m = synth.random_model((16, 16, 16, 8), (32, 32, 32, 16), 12, seed=0)
    fc, _ = bench.flops_per_point(m)
    assert fc == 74272                                # C4


def test_device_tensor_trims_library_cache_on_torch_oom(monkeypatch):
    # Gram-sized torch buffers: a torch out-of-memory error hands the
    # library's cached device blocks back (fstk_gpu_trim_device_cache) and
    # retries once.
    import torch

    from paper_1907_05884_b200 import _lib

    calls = {"empty": 0, "trim": []}
    real_empty = torch.empty

    def flaky_empty(*a, **k):
        calls["empty"] += 1
        if calls["empty"] == 1:
            raise torch.OutOfMemoryError("simulated")
        return real_empty(*a, **k)

    monkeypatch.setattr(torch, "empty", flaky_empty)
    monkeypatch.setattr(_lib, "trim_device_cache", lambda dev=-1: calls["trim"].append(dev) or 0)
    t = _lib.device_tensor(16, torch.device("cpu", 0))
    assert t.numel() == 16 and t.dtype == torch.float64
    assert calls["empty"] == 2 and len(calls["trim"]) == 1
