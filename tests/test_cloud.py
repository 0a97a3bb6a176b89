"""Point-cloud I/O (ingest.cpp:19-49, 600-754; format.md:29-55) on CPU, and
FPTC ingest to a device SoA buffer on the GPU."""
import numpy as np
import pytest

import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import synth
from paper_1907_05884_b200.cloud import PointCloud


def _pc(n=500, d=3, seed=1):
    p = synth.uniform_points(n, d, seed)
    return PointCloud.from_data(p, np.sin(p[:, 0]) * 1e-3 + np.pi * p[:, -1])


def test_fptc_round_trip_bit_exact(tmp_path):
    pc = _pc()
    pc.box_lo = pc.box_lo - 0.25      # the stored box survives (not recomputed)
    path = str(tmp_path / "c.fptc")
    F.write_cloud_binary(pc, path)
    back = F.read_cloud(path)
    assert np.array_equal(back.points, pc.points) and np.array_equal(back.values, pc.values)
    assert np.array_equal(back.box_lo, pc.box_lo) and np.array_equal(back.box_hi, pc.box_hi)
    raw = open(path, "rb").read()
    assert raw[:4] == b"FPTC" and len(raw) == 20 + 16 * 3 + 8 * 500 * 3 + 8 * 500
    # point-major payload
    assert np.array_equal(np.frombuffer(raw, "<f8", 3, 20 + 48), pc.points[0])


def test_fptc_rejects_corrupt(tmp_path):
    pc = _pc(50)
    path = tmp_path / "c.fptc"
    F.write_cloud_binary(pc, str(path))
    raw = path.read_bytes()
    for bad in (raw[:-1], raw + b"\0", b"FPTX" + raw[4:], raw[:4] + b"\2\0\0\0" + raw[8:]):
        path.write_bytes(bad)
        with pytest.raises(OSError) as e:
            F.read_cloud_binary(str(path))
        assert e.value.kind == "Decode"
    with pytest.raises(OSError) as e:
        F.read_cloud(str(tmp_path / "missing.fptc"))
    assert e.value.kind == "Io"


def test_csv_round_trip_and_points_reader(tmp_path):
    pc = _pc(40, 2)
    path = str(tmp_path / "c.csv")
    F.write_cloud_csv(pc, path)
    back = F.read_cloud(path)
    assert np.array_equal(back.points, pc.points) and np.array_equal(back.values, pc.values)
    pts = F.read_points_csv(path, 2)                     # trailing value column ignored
    assert np.array_equal(pts, pc.points)
    with pytest.raises(ValueError) as e:
        F.read_points_csv(path, 3)
    assert e.value.kind == "Parameter"
    (tmp_path / "w.csv").write_text("y0,y1,value\n1,2,3\n1,2\n")
    with pytest.raises(OSError):
        F.read_cloud_csv(str(tmp_path / "w.csv"))


def test_cloud_validation():
    p = synth.uniform_points(10, 2, 3)
    with pytest.raises(ValueError) as e:
        PointCloud.from_data(p, np.full(10, np.nan))
    assert e.value.kind == "Data"
    with pytest.raises(ValueError):
        PointCloud.from_data(np.zeros((0, 2)), np.zeros(0))


@pytest.mark.gpu
def test_fptc_to_device_soa(tmp_path):
    pc = _pc(100_003, 4, 7)
    path = str(tmp_path / "c.fptc")
    F.write_cloud_binary(pc, path)
    pts_t, vals_t, lo, hi = F.read_cloud_device(path)
    assert pts_t.shape == (4, 100_003)
    assert np.array_equal(pts_t.cpu().numpy(), np.ascontiguousarray(pc.points.T))
    assert np.array_equal(vals_t.cpu().numpy(), pc.values)
    m = synth.random_model((4, 3, 3, 2), (5, 5, 5, 5), 3, seed=1)
    assert np.array_equal(m.evaluate_device(pts_t).cpu().numpy(), m.evaluate_batch(pc.points))
