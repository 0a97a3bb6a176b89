"""GPU scattered-to-grid IDW interpolation (fstk_idw.cu) against the oracle
restatement of interpolate_to_grid (ingest.cpp:265-383): identical retained
neighbour sets (sample ids in (distance, id) order) at every node, values
within 1e-12, identical reports; the reference's own test cases
(test_ingest.cpp:115-213); errors as the reference raises them."""
import numpy as np
import pytest

import paper_1907_05884_b200 as F

pytestmark = pytest.mark.gpu


def _cloud(pts, vals, box=None):
    pc = F.PointCloud.from_data(pts, vals)
    if box is not None:
        pc.box_lo, pc.box_hi = np.asarray(box[0], float), np.asarray(box[1], float)
    return pc


def _check(O, pts, vals, sizes, intervals=None, k=0, power=2.0, box=None):
    d = pts.shape[1]
    iv = intervals or [(0.0, 1.0)] * d
    grid = F.StructuredGrid(list(sizes), iv)
    pc = _cloud(pts, vals, box)
    g, rep, nb = F.interpolate_to_grid(pc, grid, F.InterpolationOptions(k, power), return_neighbors=True)
    go, repo, nbo = O.interpolate_to_grid(pts, vals, sizes, iv, neighbors=k, power=power,
                                          box=(pc.box_lo, pc.box_hi), return_neighbors=True)
    assert g.shape == tuple(sizes)
    assert np.array_equal(nb, nbo)  # identical neighbour sets, in (d2, id) order
    err = np.abs(g - go) / np.maximum(1.0, np.abs(go))
    assert err.max() <= 1e-12, err.max()
    assert rep.box_covered == repo["box_covered"]
    assert rep.max_nearest_distance == repo["max_nearest_distance"]
    assert rep.extrapolated_fraction == repo["extrapolated_fraction"]
    return g, rep


@pytest.mark.parametrize("case", range(8))
def test_idw_matches_oracle(O, case):
    rng = np.random.default_rng(100 + case)
    d = [3, 3, 2, 1, 4, 3, 3, 2][case]
    q = [20_000, 5_000, 3_000, 400, 6_000, 30_000, 2_000, 50][case]
    sizes = [(17, 16, 15), (32, 20, 9), (40, 33), (57,), (7, 6, 5, 4), (24, 24, 24), (12, 10, 8),
             (9, 9)][case]
    k = [0, 5, 12, 0, 0, 0, 40, 3][case]
    power = [2.0, 1.5, 3.0, 2.0, 2.0, 2.0, 2.0, 0.7][case]
    if case == 5:  # clustered: half near a surface, as C3's mixture
        a = rng.random((q // 2, 3))
        b = rng.random((q - q // 2, 3))
        b[:, 2] = 0.5 + 0.05 * np.sin(2 * np.pi * b[:, 0]) + rng.uniform(-0.03, 0.03, q - q // 2)
        pts = np.vstack([a, b])
    elif case == 6:  # cloud wider than the grid box: extrapolated nodes
        pts = rng.random((q, d)) * 3.0 - 1.0
    else:
        pts = rng.random((q, d))
    vals = np.tanh((pts[:, -1] - 0.5) / 0.05) + 0.1 * rng.normal(size=q)
    iv = None
    if case == 2:
        iv = [(-0.5, 1.5), (0.25, 0.75)]
    _check(O, pts, vals, sizes, iv, k, power)


def test_idw_exact_hits_on_nodes(O):  # test_ingest.cpp:115-134
    xs = np.array([i / 4 for i in range(5)])
    ys = np.array([j / 3 for j in range(4)])
    f = lambda x, y: 3.0 * x - y + 0.25 * x * y  # noqa: E731
    pts = np.array([(x, y) for y in ys for x in xs])
    vals = f(pts[:, 0], pts[:, 1])
    g, _ = _check(O, pts, vals, (5, 4))
    for i in range(5):
        for j in range(4):
            assert g[i, j] == f(xs[i], ys[j])


def test_idw_constant_and_smooth_fields(O):  # test_ingest.cpp:136-170
    rng = np.random.default_rng(17)
    pts = rng.random((300, 2))
    g, _ = _check(O, pts, np.full(300, 2.75), (12, 9))
    assert np.abs(g - 2.75).max() <= 1e-12
    n = 50
    pts = np.random.default_rng(19).random((16 * n * n, 2))
    vals = np.sin(np.pi * pts[:, 0]) * np.cos(np.pi * pts[:, 1])
    g, rep = _check(O, pts, vals, (n, n))
    x = np.array([i / (n - 1) for i in range(n)])
    assert np.abs(g - np.sin(np.pi * x)[:, None] * np.cos(np.pi * x)[None, :]).max() <= 5e-2
    assert rep.box_covered


def test_idw_large_grid_matches_oracle(O):
    # C1's upstream step at full size: 200k points to a 64^3 grid.
    rng = np.random.default_rng(7)
    q = 200_000
    pts = rng.random((q, 3))
    x, y, z = pts.T
    vals = np.tanh((z - 0.5 - 0.05 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y)) / 0.02)
    _check(O, pts, vals, (64, 64, 64))


def test_idw_errors():
    rng = np.random.default_rng(29)
    pts = rng.random((50, 2))
    v = rng.random(50)
    grid = F.StructuredGrid.unit([4, 4])
    bad = v.copy()
    bad[10] = np.nan
    pc = F.PointCloud(np.asfortranarray(pts), bad, pts.min(0), pts.max(0))
    with pytest.raises(ValueError) as e:
        F.interpolate_to_grid(pc, grid)
    assert e.value.kind == "Data"
    pc = F.PointCloud.from_data(pts, v)
    with pytest.raises(ValueError) as e:
        F.interpolate_to_grid(pc, grid, F.InterpolationOptions(0, -1.0))
    assert e.value.kind == "Parameter"
    with pytest.raises(ValueError) as e:
        F.interpolate_to_grid(pc, F.StructuredGrid.unit([4, 4, 4]))
    assert e.value.kind == "Shape"
    with pytest.raises(ValueError) as e:
        F.interpolate_to_grid(pc, F.StructuredGrid([4, 1], [(0, 1), (0, 1)]))
    assert e.value.kind == "Parameter"
