"""Column-sharded refit (fstk_gpu_refit_begin_columns / exchange_layout /
adopt_rows): each shard transforms its columns for every row; one
all-to-all (done in-process here, as dist.exchange_columns does over NCCL)
leaves row slabs bit-identical to the row-sharded begin's, and the refit that
follows matches the oracle's QR core."""
import numpy as np
import pytest

import paper_1907_05884_b200 as F
from conftest import rel
from paper_1907_05884_b200 import synth

pytestmark = pytest.mark.gpu
CORE_TOL = 1e-9


def _data(O, model, q, seed, noise=0.01):
    pts = synth.uniform_points(q, model.order, seed)
    vals = O.evaluate_batch(model, pts) + noise * np.random.default_rng(seed).normal(size=q)
    return pts, vals


def _exchange_in_process(sessions):
    import torch

    bufs = [s.exchange_buffers() for s in sessions]
    G = len(sessions)
    for h in range(G):
        parts = []
        for g in range(G):
            send, sc, _, _ = bufs[g]
            off = sum(sc[:h])
            parts.append(send[off:off + sc[h]])
        recv, rc = bufs[h][2], bufs[h][3]
        assert [p.numel() for p in parts] == rc
        recv.copy_(torch.cat(parts))
    torch.cuda.synchronize()
    for s in sessions:
        s.adopt_rows()


@pytest.mark.parametrize("t", ["dct", "wht", "fft"])
@pytest.mark.parametrize("G", [2, 3])
def test_column_sharded_rows_are_bitexact(O, t, G):
    m = synth.random_model((5, 4, 3), [6, 6, 6], 4, seed=3)
    pts, vals = _data(O, m, 30_000, 4)
    cols = [F.RefitSession(m, pts, vals, seed=17, transform=t, shard=g, shards=G,
                           layout="columns") for g in range(G)]
    _exchange_in_process(cols)
    for g in range(G):
        r = F.RefitSession(m, pts, vals, seed=17, transform=t, shard=g, shards=G)
        ac, bc = cols[g].sketched()
        ar, br = r.sketched()
        assert ac.shape == ar.shape
        assert np.array_equal(ac, ar) and np.array_equal(bc, br)
        r.close()
    for s in cols:
        s.close()


def test_single_shard_columns_layout_equals_rows(O):
    m = synth.random_model((4, 3, 2), [6, 6, 6], 4, seed=5)
    pts, vals = _data(O, m, 20_000, 6)
    c = F.RefitSession(m, pts, vals, seed=2, layout="columns")
    _exchange_in_process([c])
    r = F.RefitSession(m, pts, vals, seed=2)
    a1, b1 = c.sketched()
    a2, b2 = r.sketched()
    assert np.array_equal(a1, a2) and np.array_equal(b1, b2)
    c.close()
    r.close()


def test_column_sharded_refit_matches_oracle(O):
    import torch

    m = synth.random_model((8, 8, 6), [8, 8, 8], 5, seed=7)
    pts, vals = _data(O, m, 60_000, 8)
    R = 8 * 8 * 6
    G = 3
    cols = [F.RefitSession(m, pts, vals, seed=9, shard=g, shards=G, layout="columns")
            for g in range(G)]
    with pytest.raises(F.FstkValueError):  # the exchange must come first
        cols[0].normal_equations(torch.empty(R * R, dtype=torch.float64, device="cuda"),
                                 torch.empty(R, dtype=torch.float64, device="cuda"))
    _exchange_in_process(cols)
    gs = [torch.empty(R * R, dtype=torch.float64, device="cuda") for _ in range(G)]
    rs = [torch.empty(R, dtype=torch.float64, device="cuda") for _ in range(G)]
    for s, g, r in zip(cols, gs, rs):
        s.normal_equations(g, r)
    gsum, rsum = sum(gs), sum(rs)
    xs = [torch.empty_like(rsum) for _ in range(G)]
    for s, x in zip(cols, xs):
        assert s.factor(gsum, rsum, x)
    for _ in range(5):
        parts = [torch.empty_like(rsum) for _ in range(G)]
        for s, x, p in zip(cols, xs, parts):
            s.correction(x, p)
        tot = sum(parts)
        for s, x in zip(cols, xs):
            s.apply(tot, x)
    core = cols[0].finish(xs[0])
    core_o, _ = O.reestimate_core(m, pts, vals, seed=9)
    assert rel(core, core_o) <= CORE_TOL
    for s in cols:
        s.close()


def test_none_transform_columns_layout_is_row_local(O):
    m = synth.random_model((4, 3, 2), [6, 6, 6], 4, seed=5)
    pts, vals = _data(O, m, 20_000, 6)
    s = F.RefitSession(m, pts, vals, seed=2, transform="none", shard=0, shards=2,
                       layout="columns")
    assert s.exchange_buffers() is None  # nothing to exchange
    r = F.RefitSession(m, pts, vals, seed=2, transform="none", shard=0, shards=2)
    a1, b1 = s.sketched()
    a2, b2 = r.sketched()
    assert np.array_equal(a1, a2) and np.array_equal(b1, b2)
    s.close()
    r.close()


@pytest.mark.parametrize("t", ["dct", "fft"])
def test_column_layout_with_thin_shards(O, t):
    # R + 1 = 7 columns and S = 8 sample rows over 5 shards: shards own one or
    # two columns and one or two rows; the exchange still lands bit-exactly.
    m = synth.random_model((3, 2, 1), [4, 4, 4], 3, seed=11)
    pts, vals = _data(O, m, 5_000, 12)
    G = 5
    cols = [F.RefitSession(m, pts, vals, seed=4, transform=t, sample_rows=8, shard=g, shards=G,
                           layout="columns") for g in range(G)]
    _exchange_in_process(cols)
    for g in range(G):
        r = F.RefitSession(m, pts, vals, seed=4, transform=t, sample_rows=8, shard=g, shards=G)
        ac, bc = cols[g].sketched()
        ar, br = r.sketched()
        assert np.array_equal(ac, ar) and np.array_equal(bc, br)
        r.close()
    for s in cols:
        s.close()


def test_column_layout_more_shards_than_columns(O):
    # 9 shards for R + 1 = 7 columns: two shards transform nothing.
    m = synth.random_model((3, 2, 1), [4, 4, 4], 3, seed=13)
    pts, vals = _data(O, m, 5_000, 14)
    G = 9
    cols = [F.RefitSession(m, pts, vals, seed=4, sample_rows=18, shard=g, shards=G,
                           layout="columns") for g in range(G)]
    _exchange_in_process(cols)
    for g in range(G):
        r = F.RefitSession(m, pts, vals, seed=4, sample_rows=18, shard=g, shards=G)
        ac, bc = cols[g].sketched()
        ar, br = r.sketched()
        assert np.array_equal(ac, ar) and np.array_equal(bc, br)
        r.close()
    for s in cols:
        s.close()


@pytest.mark.parametrize("t", ["dct", "fft"])
def test_column_sharded_rows_bitexact_at_1m(O, t):
    # q_pad = 2^20 (the warp-level first pass) with packed per-shard stores.
    m = synth.random_model((3, 2, 2), [5, 5, 5], 3, seed=13)
    pts, vals = _data(O, m, 1_150_000, 14)
    G = 2
    cols = [F.RefitSession(m, pts, vals, seed=5, transform=t, shard=g, shards=G, sample_rows=4096,
                           layout="columns") for g in range(G)]
    _exchange_in_process(cols)
    for g in range(G):
        r = F.RefitSession(m, pts, vals, seed=5, transform=t, shard=g, shards=G, sample_rows=4096)
        assert r.info_dict()["padded_rows"] == 1 << 20
        ac, bc = cols[g].sketched()
        ar, br = r.sketched()
        assert np.array_equal(ac, ar) and np.array_equal(bc, br)
        r.close()
    for s in cols:
        s.close()
