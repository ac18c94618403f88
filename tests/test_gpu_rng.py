"""GPU library pin of the oracle's RNG counter layout (reading 2; SURVEY.md §8(c) "Library pin").

cuRAND's device Philox4x32-10, initialised with curand_init(key, subsequence = v, offset = (h << 34) | j),
starts at counter {j>>2, h, lo32 v, hi32 v} with key {lo32 key, hi32 key} and returns word j & 3
first (curand_kernel.h: skipahead_sequence adds v to ctr.z/w; skipahead adds offset/4 to ctr.x/y
and keeps offset & 3).  So its first curand() must equal oracle.philox_u32(key, h, v, j) for every
tuple — over asymmetric tuples (key halves differ, h > 0, v >= 2^32, j >= 4), any swap of counter
words, of h and v, or of the key halves in the oracle fails this test.
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "curand_pin.cu")
SO = os.path.join(HERE, "native", "libcurand_pin.so")


def _lib():
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O2", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-shared", "-Xcompiler", "-fPIC", "-o", SO, SRC])
    L = ctypes.CDLL(SO)
    L.curand_pin_first.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int]
    return L


def test_oracle_philox_equals_device_curand():
    rng = np.random.default_rng(2310_00837)
    n = 4096
    key = rng.integers(0, 2**63, n, dtype=np.uint64) * 2 + 1          # both halves non-zero, distinct
    h = rng.integers(0, 2**30, n, dtype=np.uint64)                   # (h << 34) must fit 64 bits
    v = rng.integers(0, 2**63, n, dtype=np.uint64)                   # mostly >= 2^32
    j = rng.integers(0, 2**34, n, dtype=np.uint64)
    # fixed asymmetric corner cases: small values and the sampler's real ranges
    fixed = [(0x299F31D0A4093822, 1, (3 << 32) | 7, 5), (0x48454C494F53, 2, 123456789, 14),
             (1, 0, 0, 0), (0xFFFFFFFF00000001, 7, 2**32, 4), (0x9E3779B97F4A7C15, 3, 110_999_999, 31)]
    for i, (k_, h_, v_, j_) in enumerate(fixed):
        key[i], h[i], v[i], j[i] = k_, h_, v_, j_
    off = (h << np.uint64(34)) | j
    out = np.zeros(n, dtype=np.uint32)
    assert _lib().curand_pin_first(key.ctypes.data, v.ctypes.data, off.ctypes.data, out.ctypes.data, n) == 0
    exp = np.array([oracle.philox_u32(int(key[i]), int(h[i]), int(v[i]), int(j[i])) for i in range(n)], dtype=np.uint32)
    bad = np.nonzero(out != exp)[0]
    assert bad.size == 0, [(hex(int(key[i])), int(h[i]), int(v[i]), int(j[i]), hex(out[i]), hex(exp[i])) for i in bad[:5]]
