"""Pins for the oracle's Omega generator (oracle/philox.py, DESIGN reading R3)."""
import ctypes
import ctypes.util
import os

import numpy as np
import pytest
from scipy import stats

from oracle.philox import philox4x32_10, omega_rows, philox_words

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    with open(os.path.join(GOLD, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(t, 16) for t in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_random123_kat():
    kat = _kat()
    assert len(kat) == 3
    for ctr, key, out in kat:
        got = philox4x32_10([np.uint64(c) for c in ctr], [np.uint64(k) for k in key])
        assert [int(g) for g in got] == out


def _curand():
    for cand in ("/usr/local/cuda/lib64/libcurand.so", ctypes.util.find_library("curand")):
        if cand and os.path.exists(cand) or (cand and not cand.startswith("/")):
            try:
                return ctypes.CDLL(cand)
            except OSError:
                pass
    return None


@pytest.mark.parametrize("seed", [0, 2 ** 64 - 1, 12345, 0xDEADBEEF12345678])
def test_curand_host_generator(seed):
    """libcurand's HOST Philox4x32-10 generator (no GPU needed) emits block t as
    Philox(ctr=(0,0,t,0), key=seed): an implementation independent of ours."""
    lib = _curand()
    if lib is None:
        pytest.skip("libcurand not available")
    gen = ctypes.c_void_p()
    assert lib.curandCreateGeneratorHost(ctypes.byref(gen), 161) == 0  # PHILOX4_32_10
    try:
        assert lib.curandSetPseudoRandomGeneratorSeed(gen, ctypes.c_ulonglong(seed)) == 0
        n = 64
        out = (ctypes.c_uint * n)()
        assert lib.curandGenerate(gen, out, ctypes.c_size_t(n)) == 0
        ref = np.array(out[:], dtype=np.uint32).reshape(-1, 4)
        t = np.arange(ref.shape[0], dtype=np.uint64)
        z = np.zeros_like(t)
        key = (np.uint64(seed & 0xFFFFFFFF), np.uint64(seed >> 32))
        got = np.stack(philox4x32_10((z, z, t, z), key), axis=1)
        np.testing.assert_array_equal(got, ref)
    finally:
        lib.curandDestroyGenerator(gen)


def test_counter_layout_words():
    """philox_words places (j, mode|v<<8, c_lo, c_hi) in the counter (reading R3)."""
    c = np.array([0, 1, (7 << 32) + 5], dtype=np.uint64)
    w = philox_words(0x1122334455667788, 3, c, 9, v=1)
    for i, ci in enumerate(c):
        ref = philox4x32_10((np.uint64(9), np.uint64(3 | (1 << 8)), np.uint64(int(ci) & 0xFFFFFFFF),
                             np.uint64(int(ci) >> 32)), (np.uint64(0x55667788), np.uint64(0x11223344)))
        assert [int(x[i]) for x in w] == [int(r) for r in ref]


def test_box_muller_mapping_from_words():
    """Columns 4j..4j+3 are the two Box-Muller pairs of the block's 4 words: the
    squared radius of pair (k=4j, 4j+1) equals -2 ln u0 and the angle is 2 pi u1."""
    cols = np.arange(1000, dtype=np.int64)
    om = omega_rows(7, 2, cols, 8)
    for j in range(2):
        w = philox_words(7, 2, cols.astype(np.uint64), j)
        u = [(x.astype(np.float64) + 0.5) * 2.0 ** -32 for x in w]
        r2a = om[:, 4 * j] ** 2 + om[:, 4 * j + 1] ** 2
        r2b = om[:, 4 * j + 2] ** 2 + om[:, 4 * j + 3] ** 2
        np.testing.assert_allclose(r2a, -2 * np.log(u[0]), rtol=1e-13)
        np.testing.assert_allclose(r2b, -2 * np.log(u[2]), rtol=1e-13)
        ang = np.mod(np.arctan2(om[:, 4 * j + 1], om[:, 4 * j]), 2 * np.pi)
        np.testing.assert_allclose(ang, 2 * np.pi * u[1], atol=1e-9)


def test_gaussian_statistics():
    """i.i.d. N(0,1): KS test against scipy's normal CDF, mean/var bounds
    (mean +-0.02, var +-0.05 on 1e5 samples), no cross-column correlation."""
    om = omega_rows(0, 0, np.arange(25000, dtype=np.int64), 8)
    z = om.ravel()
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1) < 0.05
    assert stats.kstest(z, "norm").pvalue > 1e-3
    cc = np.corrcoef(om.T)
    assert np.max(np.abs(cc - np.eye(8))) < 0.05
    # different modes / seeds / draw types are different streams
    om2 = omega_rows(0, 1, np.arange(25000, dtype=np.int64), 8)
    om3 = omega_rows(1, 0, np.arange(25000, dtype=np.int64), 8)
    om4 = omega_rows(0, 0, np.arange(25000, dtype=np.int64), 8, v=1)
    for o in (om2, om3, om4):
        assert abs(np.corrcoef(om.ravel(), o.ravel())[0, 1]) < 0.02


def test_partition_and_block_invariance():
    """Counter-based: any row subset / column window equals the corresponding part of
    the full matrix (sharding and adaptive blocks draw the same Omega)."""
    full = omega_rows(3, 1, np.arange(500, dtype=np.int64), 23)
    rows = np.array([499, 3, 77, 250], dtype=np.int64)
    np.testing.assert_array_equal(omega_rows(3, 1, rows, 23), full[rows])
    np.testing.assert_array_equal(omega_rows(3, 1, np.arange(500), 7, k0=5), full[:, 5:12])
    np.testing.assert_array_equal(omega_rows(3, 1, np.arange(500), 1, k0=22), full[:, 22:23])
