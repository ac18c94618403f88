"""CPU oracle for the Helios mini-batch preparation path — TEST INFRASTRUCTURE ONLY.

Plain, slow, single-threaded C++ (``oracle/oracle.cpp``), loaded through ctypes.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package; the product path (``paper_2310_00837_b200``) never does.

Each function cites the passage it follows in ``oracle.cpp``'s header.  Every function is pinned
by ``tests/test_oracle_*.py`` (``-m "not gpu"``) against something other than itself; there is no
"parity unpinned" function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

TIER_HBM, TIER_HOST, TIER_FILE = 0, 1, 2
OK, E_INVALID, E_RANGE, E_CAPACITY, E_NOMEM, E_CUDA, E_IO = range(7)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _SO, src])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i64, u64, i32, u32, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_void_p
        L.oracle_philox4x32_10.argtypes = [vp, vp, vp]
        L.oracle_philox_u32.restype = u32
        L.oracle_philox_u32.argtypes = [u64, i32, i64, i64]
        L.oracle_floyd.argtypes = [i64, i64, vp, vp]
        L.oracle_sample_row.restype = i64
        L.oracle_sample_row.argtypes = [u64, i32, i64, i64, i64, vp]
        L.oracle_sample.restype = ctypes.c_int
        L.oracle_sample.argtypes = [i64, vp, vp, vp, i64, vp, i32, u64, i64, vp, vp, vp, i64, vp, i64, vp]
        L.oracle_presample.restype = ctypes.c_int
        L.oracle_presample.argtypes = [i64, vp, vp, vp, vp, i64, vp, vp, i32, vp]
        L.oracle_cache_dir.restype = ctypes.c_int
        L.oracle_cache_dir.argtypes = [i64, vp, i32, i64, i64, i32, vp, vp]
        L.oracle_lookup_counts.argtypes = [vp, vp, i64, i32, vp]
        L.oracle_gather.restype = ctypes.c_int
        L.oracle_gather.argtypes = [vp, i64, i32, vp, ctypes.c_char_p, i64, i64, vp, vp]
        _lib = L
    return _lib


def _p(a) -> int | None:
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def philox4x32_10(ctr, key) -> list[int]:
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(o))
    return [int(x) for x in o]


def philox_u32(key: int, h: int, v: int, j: int) -> int:
    return int(lib().oracle_philox_u32(key & 0xFFFFFFFFFFFFFFFF, h, v, j))


def floyd(d: int, k: int, t) -> list[int]:
    t = _c(t, np.uint32)
    P = np.zeros(max(1, k), dtype=np.int64)
    lib().oracle_floyd(d, k, _p(t), _p(P))
    return [int(x) for x in P[:k]]


def sample_row(key: int, h: int, v: int, d: int, f: int) -> list[int]:
    P = np.zeros(max(1, d), dtype=np.int64)
    k = lib().oracle_sample_row(key & 0xFFFFFFFFFFFFFFFF, h, v, d, f, _p(P))
    return [int(x) for x in P[:k]]


@dataclass
class Batch:
    nodes: np.ndarray                 # int64[n_L]
    level_counts: np.ndarray          # int64[L+1]
    edge_counts: np.ndarray           # int64[L]
    block_indptr: list = field(default_factory=list)   # L x int32[n_h+1]
    block_indices: list = field(default_factory=list)  # L x int32[e_h]


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: status {code}")
        self.code = code


def sample_bounds(n_seeds: int, fanouts, V: int, E: int) -> tuple[int, list[int]]:
    n, edges = n_seeds, []
    for f in fanouts:
        e = E if f < 0 else min(n * f, E)
        edges.append(e)
        n = min(V, n + e)
    return n, edges


def sample(indptr: np.ndarray, indices: np.ndarray, seeds, fanouts, key: int) -> Batch:
    indptr = _c(indptr, np.int64)
    indices = _c(indices, np.int32)
    V = len(indptr) - 1
    E = int(indptr[-1])
    seeds = _c(seeds, np.int64)
    fan = _c(fanouts, np.int32)
    L = len(fan)
    ncap, ecaps = sample_bounds(len(seeds), list(fan), V, E)
    # the n_h bounds for the indptr capacity
    n, bpcap = len(seeds), 0
    for h in range(L):
        bpcap += n + 1
        n = min(V, n + ecaps[h])
    nodes = np.zeros(max(1, ncap), dtype=np.int64)
    lc = np.zeros(L + 1, dtype=np.int64)
    ec = np.zeros(max(1, L), dtype=np.int64)
    bp = np.zeros(max(1, bpcap), dtype=np.int32)
    bi = np.zeros(max(1, sum(ecaps)), dtype=np.int32)
    rc = lib().oracle_sample(V, _p(indptr), _p(indices), _p(seeds), len(seeds), _p(fan), L, key & 0xFFFFFFFFFFFFFFFF,
                             len(nodes), _p(nodes), _p(lc), _p(ec), len(bp), _p(bp), len(bi), _p(bi))
    if rc != OK:
        raise OracleError(rc, "oracle_sample")
    out = Batch(nodes[: lc[L]].copy(), lc, ec[:L].copy())
    bo = eo = 0
    for h in range(L):
        nh, eh = int(lc[h]), int(ec[h])
        out.block_indptr.append(bp[bo:bo + nh + 1].copy())
        out.block_indices.append(bi[eo:eo + eh].copy())
        bo += nh + 1
        eo += eh
    return out


def presample(indptr, indices, batches: list, keys: list, fanouts) -> np.ndarray:
    indptr = _c(indptr, np.int64)
    indices = _c(indices, np.int32)
    V = len(indptr) - 1
    seeds = _c(np.concatenate(batches) if batches else np.zeros(0), np.int64)
    offs = _c(np.concatenate([[0], np.cumsum([len(b) for b in batches])]), np.int64)
    ks = _c(keys, np.uint64)
    fan = _c(fanouts, np.int32)
    hot = np.zeros(V, dtype=np.uint64)
    rc = lib().oracle_presample(V, _p(indptr), _p(indices), _p(seeds), _p(offs), len(batches), _p(ks), _p(fan), len(fan),
                                _p(hot))
    if rc != OK:
        raise OracleError(rc, "oracle_presample")
    return hot


def cache_dir(hot: np.ndarray, G: int, H: int, S: int, host_slot_is_id: bool = False) -> tuple[np.ndarray, np.ndarray]:
    hot = _c(hot, np.uint64)
    V = len(hot)
    d = np.zeros(V, dtype=np.int64)
    order = np.zeros(V, dtype=np.int64)
    rc = lib().oracle_cache_dir(V, _p(hot), G, H, S, int(host_slot_is_id), _p(d), _p(order))
    if rc != OK:
        raise OracleError(rc, "oracle_cache_dir")
    return d, order


def dir_decode(w) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(tier, owner, slot) arrays from directory words (D11 layout)."""
    u = np.asarray(w, dtype=np.int64).view(np.uint64)
    return (u >> np.uint64(62)).astype(np.int64), ((u >> np.uint64(56)) & np.uint64(63)).astype(np.int64), \
        (u & np.uint64((1 << 56) - 1)).astype(np.int64)


def lookup_counts(dir_: np.ndarray, nodes: np.ndarray, rank: int = 0) -> np.ndarray:
    dir_ = _c(dir_, np.int64)
    nodes = _c(nodes, np.int64)
    c = np.zeros(4, dtype=np.int64)
    lib().oracle_lookup_counts(_p(dir_), _p(nodes), len(nodes), rank, _p(c))
    return c


def gather(nodes, R: int, table: np.ndarray | None = None, path: str | None = None, header: int = 0,
           stride: int = 0, dir_: np.ndarray | None = None, out: np.ndarray | None = None) -> np.ndarray:
    nodes = _c(nodes, np.int64)
    if out is None:
        out = np.empty((len(nodes), R), dtype=np.uint8)
    if table is not None:
        assert table.flags.c_contiguous
    if dir_ is not None:
        dir_ = _c(dir_, np.int64)
    rc = lib().oracle_gather(_p(nodes), len(nodes), R, _p(table), (path or "").encode(), header, stride, _p(dir_),
                             _p(out))
    if rc != OK:
        raise OracleError(rc, "oracle_gather")
    return out
