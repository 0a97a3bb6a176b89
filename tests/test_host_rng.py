"""The library's host replay of the reference RNG (fstk_refit.cu: partial
Fisher-Yates with O(k) state, bitmap or comparison sort; make_plan) -- the
sampled-index stream the whole refit depends on -- checked bit-exactly on
the CPU (no GPU needed: pure host code behind the C-ABI) against the golden
vectors from the reference's own rng.cpp and, where oracle/_ref is built,
against that compiled reference over a sweep of (n, k)."""
import ctypes as C

import numpy as np
import pytest

from paper_1907_05884_b200._lib import Err, lib


def _swr(seed, n, k):
    out = np.zeros(min(n, k), dtype=np.uint64)
    err = Err()
    rc = lib().fstk_gpu_sample_without_replacement(
        C.c_uint64(seed), C.c_uint64(n), C.c_uint64(k),
        out.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(err))
    assert rc == 0, err.message
    return out


def _plan(q_w, s, seed):
    q_pad = 1
    while q_pad < q_w:
        q_pad <<= 1
    signs = np.zeros(q_pad)
    rows = np.zeros(s, dtype=np.uint64)
    scale = C.c_double()
    qp = C.c_uint64()
    err = Err()
    rc = lib().fstk_gpu_make_plan(C.c_uint64(q_w), C.c_uint64(s), C.c_uint64(seed),
                                  signs.ctypes.data_as(C.POINTER(C.c_double)),
                                  rows.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(scale),
                                  C.byref(qp), C.byref(err))
    assert rc == 0, err.message
    assert qp.value == q_pad
    return signs, rows, scale.value


def test_sample_without_replacement_matches_golden(golden):
    i = 0
    while f"swr_{i}" in golden.files:
        seed, n, k = (int(v) for v in golden[f"swr_{i}_args"])
        assert np.array_equal(_swr(seed, n, k), golden[f"swr_{i}"]), (seed, n, k)
        i += 1
    assert i >= 6


def test_make_plan_matches_golden(golden):
    i = 0
    while f"plan_{i}_rows" in golden.files:
        q_pad, s, seed = (int(v) for v in golden[f"plan_{i}_args"])
        signs, rows, scale = _plan(q_pad, s, seed)
        assert np.array_equal(np.packbits(signs < 0), golden[f"plan_{i}_negbits"])
        assert np.array_equal(rows, golden[f"plan_{i}_rows"])
        assert scale == np.sqrt(q_pad / s)
        i += 1
    assert i >= 3


# Both sides of the bitmap/sort switch (n / 64 <= 16 k), the k >= n shortcut,
# k = 0, k = n - 1, tiny and large n.
SWEEP = [(1, 1, 0), (1, 1, 1), (2, 5, 4), (3, 100, 99), (4, 1000, 1000), (5, 1000, 5000),
         (6, 1_000_000, 100), (7, 1_000_000, 977), (8, 1_000_000, 1_000), (9, 1 << 20, 1 << 18),
         (10, 16_777_216, 100_000), (11, 16_677_216, 1 << 20), (12, 123_457, 1)]


@pytest.mark.parametrize("seed,n,k", SWEEP)
def test_sample_without_replacement_matches_compiled_reference(O, seed, n, k):
    R = O.ref()
    if R is None:
        pytest.skip("oracle/_ref not built (reference tree absent)")
    want = np.zeros(min(n, k), dtype=np.uint64)
    R.ref_sample_without_replacement(C.c_uint64(seed), C.c_uint64(n), C.c_uint64(k),
                                     want.ctypes.data_as(C.POINTER(C.c_uint64)))
    got = _swr(seed, n, k)
    assert np.array_equal(got, want)
    assert np.all(np.diff(got.astype(np.int64)) > 0)  # sorted, distinct


def test_make_plan_c2_matches_oracle(O):
    q_w, s = 1 << 20, 262_144
    seed = O.mix_seed(0, 0x736B6574)
    signs, rows, scale = _plan(q_w, s, seed)
    s2, r2, sc2 = O.make_plan(q_w, s, seed)
    assert np.array_equal(signs, s2) and np.array_equal(rows, r2) and scale == sc2
