"""Pins for the oracle's RNG and subset algorithm (readings 2-3).

* Philox4x32-10 against the Random123 known-answer vectors (tests/golden/philox_kat.txt).
* Floyd's algorithm by exhaustive enumeration: over every draw sequence t_j in [0, d-k+j], each
  k-subset of [0, d) appears exactly k! times (Bentley & Floyd 1987) — brute force, d <= 7.
* Sampling a row with real Philox draws: marginal inclusion frequency k/d (SPEC.md:333 idea:
  0.25 +- 0.01 at d=100, k=25) and a chi-square test over all C(d,k) subsets for small d.
"""
import itertools
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,expect", _kat())
def test_philox_kat(ctr, key, expect):
    assert oracle.philox4x32_10(ctr, key) == expect


def test_philox_u32_counter_layout():
    """Reading 2's counter layout {j>>2, h, lo32 v, hi32 v}, key {lo32 key, hi32 key}, word j&3,
    pinned on the ASYMMETRIC Random123 KAT block (ctr = 243f6a88 85a308d3 13198a2e 03707344,
    key = a4093822 299f31d0): every counter / key word differs, so swapping any two counter words,
    h with lo32(v), or the key halves, or taking another output word, changes the result."""
    ctr, key, expect = _kat()[2]
    assert len(set(ctr)) == 4 and key[0] != key[1]
    k64 = (key[1] << 32) | key[0]
    h = ctr[1] - (1 << 32) if ctr[1] >= 1 << 31 else ctr[1]   # int32 hop index carrying the word 0x85a308d3
    v = (ctr[3] << 32) | ctr[2]
    got = [oracle.philox_u32(k64, h, v, (ctr[0] << 2) | w) for w in range(4)]
    assert got == expect
    # a permuted call must not reproduce it (the test can tell the fields apart)
    assert [oracle.philox_u32(k64, ctr[2], (ctr[3] << 32) | ctr[1], (ctr[0] << 2) | w) for w in range(4)] != expect
    # symmetric KATs too (ctr = 0 / all-ones)
    assert [oracle.philox_u32(0, 0, 0, j) for j in range(4)] == _kat()[0][2]
    assert [oracle.philox_u32(0xFFFFFFFFFFFFFFFF, -1, -1, (0xFFFFFFFF << 2) | j) for j in range(4)] == _kat()[1][2]


def _host_curand_philox(seed: int, n: int):
    """n outputs of cuRAND's HOST Philox4x32-10 generator (libcurand, a library independent of the
    oracle), or None when libcurand is not available."""
    import ctypes
    import glob
    libs = (glob.glob("/usr/local/cuda/lib64/libcurand.so*")
            + glob.glob(os.path.join(os.path.dirname(np.__file__), "..", "nvidia", "curand", "lib", "libcurand.so*")))
    if not libs:
        return None
    cr = ctypes.CDLL(sorted(libs)[0])
    g = ctypes.c_void_p()
    CURAND_RNG_PSEUDO_PHILOX4_32_10 = 161
    assert cr.curandCreateGeneratorHost(ctypes.byref(g), CURAND_RNG_PSEUDO_PHILOX4_32_10) == 0
    try:
        assert cr.curandSetPseudoRandomGeneratorSeed(g, ctypes.c_ulonglong(seed)) == 0
        out = np.zeros(n, dtype=np.uint32)
        assert cr.curandGenerate(g, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(n)) == 0
    finally:
        cr.curandDestroyGenerator(g)
    return out


def test_philox_u32_vs_host_curand():
    """Library pin of the key and vertex words: cuRAND's host Philox4x32-10 generator with seed s emits,
    as its i-th block of 4 outputs, Philox(ctr = {0, 0, i, 0}, key = {lo32 s, hi32 s}) (one
    subsequence per block; checked for the first 4096 blocks), which is philox_u32(s, h=0, v=i, j=0..3)
    under reading 2.  The hop and slot-block words are pinned by the GPU test against
    curand_init(key, v, (h << 34) | j) (tests/test_gpu_rng.py) and by the asymmetric KAT above."""
    seed = 0x299F31D0A4093822
    n_blocks = 4096
    out = _host_curand_philox(seed, 4 * n_blocks)
    if out is None:
        pytest.skip("libcurand not found")
    for i in list(range(64)) + [255, 256, 1000, 4095]:
        assert [oracle.philox_u32(seed, 0, i, j) for j in range(4)] == [int(x) for x in out[4 * i: 4 * i + 4]], i


@pytest.mark.parametrize("d", range(1, 8))
def test_floyd_exhaustive(d):
    for k in range(0, d + 1):
        counts = {}
        ranges = [range(d - k + j + 1) for j in range(k)]
        for t in itertools.product(*ranges):
            P = oracle.floyd(d, k, list(t))
            assert len(set(P)) == k and all(0 <= p < d for p in P)
            key = tuple(sorted(P))
            counts[key] = counts.get(key, 0) + 1
        assert len(counts) == math.comb(d, k)
        assert set(counts.values()) == {math.factorial(k)}


def test_sample_row_take_all_and_bounds():
    assert oracle.sample_row(1, 0, 5, 3, 10) == [0, 1, 2]        # deg <= fanout: all, CSR order
    assert oracle.sample_row(1, 0, 5, 0, 10) == []               # isolated
    assert oracle.sample_row(1, 0, 5, 40, -1) == list(range(40))  # fanout -1: all
    P = oracle.sample_row(7, 2, 123, 10**6, 15)                   # hub: exactly 15 distinct positions
    assert len(P) == 15 and len(set(P)) == 15 and all(0 <= p < 10**6 for p in P)


def test_sample_row_marginal_frequency():
    d, k, trials = 100, 25, 20000
    hits = np.zeros(d)
    for key in range(trials):
        for p in oracle.sample_row(key * 0x9E3779B97F4A7C15 + 1, 0, 42, d, k):
            hits[p] += 1
    freq = hits / trials
    # binomial sd = sqrt(.25*.75/20000) = .0031 -> 0.25 +- 0.015 is ~5 sd
    assert np.all(np.abs(freq - 0.25) < 0.015), (freq.min(), freq.max())


def test_sample_row_subset_chi_square():
    from scipy.stats import chisquare
    d, k, trials = 6, 3, 24000
    subsets = {s: 0 for s in itertools.combinations(range(d), k)}
    for key in range(trials):
        subsets[tuple(sorted(oracle.sample_row(key + 12345, 1, 7, d, k)))] += 1
    _, p = chisquare(list(subsets.values()))
    assert p > 1e-4
