"""Oracle pins for the IDW interpolation restatement (oracle/fstk_oracle.cpp,
ingest.cpp:117-383): the reference's own tests (test_ingest.cpp:115-213)
restated, plus a brute-force check of the retained neighbour sets.  CPU only
-- the oracle is the checker of fstk_idw.cu (tests/test_gpu_idw.py)."""
import numpy as np
import pytest

from oracle import oracle as O


def test_exact_values_when_samples_sit_on_nodes():  # test_ingest.cpp:115-134
    xs, ys = np.linspace(0, 1, 5), np.linspace(0, 1, 4)
    xs = np.array([0.0 + 1.0 * i / 4 for i in range(5)])
    ys = np.array([0.0 + 1.0 * j / 3 for j in range(4)])
    f = lambda x, y: 3.0 * x - y + 0.25 * x * y  # noqa: E731
    pts = np.array([(x, y) for y in ys for x in xs])
    vals = f(pts[:, 0], pts[:, 1])
    g, _ = O.interpolate_to_grid(pts, vals, (5, 4))
    for i in range(5):
        for j in range(4):
            assert g[i, j] == f(xs[i], ys[j])


def test_reproduces_constants():  # test_ingest.cpp:136-142
    rng = np.random.default_rng(17)
    pts = rng.random((300, 2))
    g, _ = O.interpolate_to_grid(pts, np.full(300, 2.75), (12, 9))
    assert np.abs(g - 2.75).max() <= 1e-12


def test_dense_smooth_cloud_small_node_error():  # test_ingest.cpp:144-170
    n = 50
    rng = np.random.default_rng(19)
    pts = rng.random((16 * n * n, 2))
    vals = np.sin(np.pi * pts[:, 0]) * np.cos(np.pi * pts[:, 1])
    g, rep = O.interpolate_to_grid(pts, vals, (n, n))
    x = np.array([i / (n - 1) for i in range(n)])
    want = np.sin(np.pi * x)[:, None] * np.cos(np.pi * x)[None, :]
    assert np.abs(g - want).max() <= 5e-2
    assert rep["box_covered"]


def test_linear_field_within_two_percent():  # test_ingest.cpp:172-201
    n, per = 20, 32
    rng = np.random.default_rng(23)
    a, b = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    base = np.stack([a.ravel(), b.ravel()], axis=1).repeat(per, axis=0)
    pts = (base + rng.random(base.shape)) / n
    vals = 2.0 * pts[:, 0] - 0.5 * pts[:, 1] + 1.0
    g, _ = O.interpolate_to_grid(pts, vals, (n, n))
    x = np.array([i / (n - 1) for i in range(n)])
    want = 2.0 * x[:, None] - 0.5 * x[None, :] + 1.0
    assert np.abs(g - want).max() <= 0.02 * 2.5


def test_nonfinite_values_rejected():  # test_ingest.cpp:203-211
    rng = np.random.default_rng(29)
    pts = rng.random((50, 2))
    v = rng.random(50)
    v[10] = np.nan
    with pytest.raises(O.OracleError) as e:
        O.interpolate_to_grid(pts, v, (4, 4))
    assert e.value.kind == "Data"
    with pytest.raises(O.OracleError) as e:
        O.interpolate_to_grid(pts, rng.random(50), (4, 4), power=0.0)
    assert e.value.kind == "Parameter"


@pytest.mark.parametrize("d,k", [(2, 0), (3, 0), (3, 11), (1, 3)])
def test_neighbour_sets_are_the_k_nearest(d, k):
    # Random data has no distance ties, so the reference's ring scan with its
    # stop rule must retain exactly the k nearest samples (brute force).
    rng = np.random.default_rng(40 + d + k)
    q = 700
    pts = rng.random((q, d)) * 1.2 - 0.1  # cloud box beyond the grid box
    vals = rng.normal(size=q)
    sizes = (9, 7, 5)[:d]
    g, rep, nb = O.interpolate_to_grid(pts, vals, sizes, neighbors=k, return_neighbors=True)
    kk = k if k > 0 else 2 * d + 2
    nodes = np.stack(np.meshgrid(*[np.array([i / (s - 1) for i in range(s)]) for s in sizes],
                                 indexing="ij"), axis=-1).reshape(-1, d, order="F")
    for node, row in zip(nodes, nb):
        d2 = ((pts - node) ** 2).sum(axis=1)
        want = np.lexsort((np.arange(q), d2))[:kk]
        assert list(row) == list(want)
    assert not rep["box_covered"]
