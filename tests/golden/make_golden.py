"""Generates tests/golden/ref_vectors.npz from the REFERENCE's own sources.

oracle/_ref/libfstk_ref.so is /root/reference/proj/src/{rng,transforms,
parallel}.cpp compiled as-is (oracle/Makefile).  These vectors pin the oracle
restatement (and, through it, the GPU path) to the reference bit for bit:

  * mix_seed / raw mt19937_64 streams / uniform_index (rng.cpp:11-61)
  * sample_without_replacement (rng.cpp:36-53), including k >= n
  * make_plan streams: q_pad signs then the sorted sample (randls.cpp:61-75)
  * fft_pow2 / unitary_fft / dct2_orthonormal / wht_orthonormal
    (transforms.cpp:26-104) on seeded inputs, n = 1 .. 2^12
  * next_pow2 boundary values (test_transforms.cpp:80-90)

Run:  make -C oracle && python tests/golden/make_golden.py
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

U64P = C.POINTER(C.c_uint64)
DP = C.POINTER(C.c_double)


def main():
    R = O.ref()
    if R is None:
        raise SystemExit("oracle/_ref/libfstk_ref.so missing (needs /root/reference; run make -C oracle)")
    out = {}
    tags = [0x76616C69, 0x73756273, 0x736B6574]
    seeds = [0, 1, 17, 99, 2**63 + 5]
    out["mix_seed_in"] = np.array([[s, t] for s in seeds for t in tags], dtype=np.uint64)
    out["mix_seed_out"] = np.array([R.ref_mix_seed(int(s), int(t)) for s in seeds for t in tags],
                                   dtype=np.uint64)
    a = np.zeros(64, dtype=np.uint64)
    R.ref_u64_stream(C.c_uint64(5489), C.c_uint64(64), a.ctypes.data_as(U64P))
    out["u64_stream_5489"] = a
    ui = np.zeros(200, dtype=np.uint64)
    assert R.ref_uniform_index_stream(C.c_uint64(3), C.c_uint64(1000003), C.c_uint64(200),
                                      ui.ctypes.data_as(U64P)) == 0
    out["uniform_index_3_1000003"] = ui
    sw_cases = [(1, 10, 3), (7, 100, 100), (7, 100, 150), (42, 1000, 37), (99, 200000, 10000),
                (O.mix_seed(0, 0x76616C69), 200000, 10000)]
    for i, (seed, n, k) in enumerate(sw_cases):
        v = np.zeros(min(n, k), dtype=np.uint64)
        R.ref_sample_without_replacement(C.c_uint64(seed), C.c_uint64(n), C.c_uint64(k),
                                         v.ctypes.data_as(U64P))
        out[f"swr_{i}_args"] = np.array([seed, n, k], dtype=np.uint64)
        out[f"swr_{i}"] = v
    plan_cases = [(32, 32, 5), (262144, 16384, O.mix_seed(0, 0x736B6574)), (1024, 40, 9)]
    for i, (q_pad, s, seed) in enumerate(plan_cases):
        sg = np.zeros(q_pad)
        rows = np.zeros(s, dtype=np.uint64)
        R.ref_plan_stream(C.c_uint64(seed), C.c_uint64(q_pad), C.c_uint64(s), sg.ctypes.data_as(DP),
                          rows.ctypes.data_as(U64P))
        out[f"plan_{i}_args"] = np.array([q_pad, s, seed], dtype=np.uint64)
        out[f"plan_{i}_negbits"] = np.packbits(sg < 0)  # compact sign record
        out[f"plan_{i}_rows"] = rows
    rng = np.random.default_rng(2024)
    for n in (1, 2, 8, 64, 1024, 4096):
        x = rng.normal(size=n)
        out[f"x_{n}"] = x
        y = x.copy()
        assert R.ref_dct2(y.ctypes.data_as(DP), C.c_uint64(n)) == 0
        out[f"dct_{n}"] = y
        y = x.copy()
        assert R.ref_wht(y.ctypes.data_as(DP), C.c_uint64(n)) == 0
        out[f"wht_{n}"] = y
        z = (x + 1j * rng.normal(size=n)).astype(np.complex128)
        out[f"z_{n}"] = z
        for inv in (0, 1):
            w = z.copy()
            assert R.ref_fft_pow2(w.ctypes.data_as(DP), C.c_uint64(n), C.c_int(inv)) == 0
            out[f"fft{inv}_{n}"] = w
            w = z.copy()
            assert R.ref_unitary_fft(w.ctypes.data_as(DP), C.c_uint64(n), C.c_int(inv)) == 0
            out[f"ufft{inv}_{n}"] = w
    np2 = [0, 1, 2, 3, 4, 5, 1023, 1024, 1025, 190000, 1000000]
    out["next_pow2_in"] = np.array(np2, dtype=np.uint64)
    out["next_pow2_out"] = np.array([R.ref_next_pow2(v) for v in np2], dtype=np.uint64)
    path = os.path.join(HERE, "ref_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
