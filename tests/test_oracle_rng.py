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
    # word j&3 of the block whose counter is {j>>2, h, lo32(v), hi32(v)}: checked on the KAT block
    # (ctr = 0, key = 0 -> 6627e8d5 e169c58d bc57ac4c 9b00dbd8), i.e. key 0, hop 0, vertex 0, j = 0..3
    expect = _kat()[0][2]
    assert [oracle.philox_u32(0, 0, 0, j) for j in range(4)] == expect
    # all-ones KAT: ctr = {ffffffff x4}, key = ffffffff x2 -> j>>2 = 0xffffffff, h = -1, v = -1
    expect1 = _kat()[1][2]
    assert [oracle.philox_u32(0xFFFFFFFFFFFFFFFF, -1, -1, (0xFFFFFFFF << 2) | j) for j in range(4)] == expect1


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
