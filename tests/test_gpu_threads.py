"""The C-ABI is callable from several host threads at once (reference:
`parallel.hpp:8-10`, the model is shareable across threads).  Concurrent
refits of different models and concurrent evaluations of one model on the
same device give exactly the sequential results."""
import threading

import numpy as np
import pytest

import paper_1907_05884_b200 as F
from paper_1907_05884_b200 import synth

pytestmark = pytest.mark.gpu


def _run_threads(fns):
    out, errs = [None] * len(fns), []

    def wrap(i, f):
        try:
            out[i] = f()
        except Exception as e:  # noqa: BLE001 - surfaced below
            errs.append(e)

    ts = [threading.Thread(target=wrap, args=(i, f)) for i, f in enumerate(fns)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    return out


def test_concurrent_refits_match_sequential():
    models = [synth.random_model((8, 8, 6), (8, 8, 8), 5, seed=60 + k) for k in range(3)]
    pts = synth.uniform_points(40_000, 3, seed=61)
    vals = synth.flame_field(pts, seed=62)
    seq = [F.reestimate_core(m, pts, vals, seed=3)[0].core for m in models]
    par = _run_threads([lambda m=m: F.reestimate_core(m, pts, vals, seed=3)[0].core for m in models])
    for a, b in zip(seq, par):
        assert np.array_equal(a, b)


def test_concurrent_evaluations_of_one_model_match():
    m = synth.random_model((12, 10, 8), (16, 16, 16), 6, seed=63)
    clouds = [synth.uniform_points(300_000, 3, seed=64 + k) for k in range(4)]
    seq = [m.evaluate_batch(p) for p in clouds]
    par = _run_threads([lambda p=p: m.evaluate_batch(p) for p in clouds])
    for a, b in zip(seq, par):
        assert np.array_equal(a, b)
