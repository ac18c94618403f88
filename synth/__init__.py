"""Seeded synthetic inputs shared by the oracle and the CUDA path (no method arithmetic here).

Generates, deterministically from a 64-bit seed:
  * a power-law CSR graph whose degree law is the Graph500 R-MAT marginal (``graph``),
  * canonical fp32 feature rows  row(v)[j] = (mix64(v*dim+j) >> 40) * 2^-24  (``features``),
  * the feature file (header + 512 B-padded rows),
  * the 1% training set, per-epoch seed batches and 64-bit batch keys.

Recipe and its citations: DESIGN.md "Input recipe" / SURVEY.md §8(d).  The C++ generator is
``synth/gen.cpp``; it is compiled on first use (plain g++, seconds).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_lib = None

HELIOS_SEED = 0x48454C494F53  # "HELIOS"


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", "-o", _SO, src])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i64, u64, i32, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p
        L.synth_mix64.restype = u64
        L.synth_mix64.argtypes = [u64]
        L.synth_perm_fwd.restype = u64
        L.synth_perm_fwd.argtypes = [ctypes.c_int, u64, u64]
        L.synth_perm_inv.restype = u64
        L.synth_perm_inv.argtypes = [ctypes.c_int, u64, u64]
        L.synth_graph_degrees.restype = i64
        L.synth_graph_degrees.argtypes = [i64, i64, u64, ctypes.c_double, vp]
        L.synth_graph_fill.argtypes = [i64, u64, ctypes.c_double, vp, vp, vp]
        L.synth_graph_compact.argtypes = [i64, vp, vp, vp, vp]
        L.synth_features.argtypes = [i64, i64, i32, vp]
        L.synth_features_at.argtypes = [vp, i64, i32, vp]
        L.synth_write_feature_file.restype = ctypes.c_int
        L.synth_write_feature_file.argtypes = [ctypes.c_char_p, i64, i32, i64, i64]
        L.synth_train_set.restype = i64
        L.synth_train_set.argtypes = [i64, u64, i32, vp]
        L.synth_epoch_order.argtypes = [vp, i64, u64, i64, vp]
        L.synth_batch_key.restype = u64
        L.synth_batch_key.argtypes = [u64, i64, i64]
        L.synth_set_threads.argtypes = [ctypes.c_int]
        L.synth_get_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def set_threads(t: int) -> None:
    lib().synth_set_threads(int(t))


def mix64(x: int) -> int:
    return int(lib().synth_mix64(x & 0xFFFFFFFFFFFFFFFF))


@dataclass
class Graph:
    V: int
    indptr: np.ndarray   # int64[V+1]
    indices: np.ndarray  # int32[E]

    @property
    def E(self) -> int:
        return int(self.indptr[-1])

    def degree_stats(self) -> dict:
        deg = np.diff(self.indptr)
        top = max(1, self.V // 100)
        # endpoint share of the top-1% vertices by in-degree (SPEC.md:508 reports skew like this)
        indeg = np.bincount(self.indices, minlength=self.V)
        share = float(np.sort(indeg)[::-1][:top].sum()) / max(1, self.E)
        return {"V": self.V, "E": self.E, "avg_deg": self.E / self.V, "max_out_deg": int(deg.max()),
                "max_in_deg": int(indeg.max()), "top1pct_in_share": round(share, 4)}


def graph(V: int, E_target: int, seed: int = HELIOS_SEED, p1: float = 0.24) -> Graph:
    """Power-law CSR: out-degrees and destinations follow the R-MAT (.57,.19,.19,.05) marginals
    over a seeded vertex permutation; self-loops and duplicate (src,dst) pairs removed."""
    L = lib()
    deg = np.empty(V, dtype=np.int64)
    tot = L.synth_graph_degrees(V, E_target, seed, p1, _p(deg))
    if tot < 0:
        raise ValueError("bad graph parameters")
    prov_indptr = np.zeros(V + 1, dtype=np.int64)
    np.cumsum(deg, out=prov_indptr[1:])
    del deg
    prov = np.empty(max(1, tot), dtype=np.int32)
    flen = np.empty(V, dtype=np.int64)
    L.synth_graph_fill(V, seed, p1, _p(prov_indptr), _p(prov), _p(flen))
    indptr = np.zeros(V + 1, dtype=np.int64)
    np.cumsum(flen, out=indptr[1:])
    del flen
    indices = np.empty(max(1, int(indptr[-1])), dtype=np.int32)
    L.synth_graph_compact(V, _p(prov_indptr), _p(prov), _p(indptr), _p(indices))
    return Graph(V, indptr, indices[: int(indptr[-1])])


def features(V: int, dim: int, out: np.ndarray | None = None, v0: int = 0) -> np.ndarray:
    """Canonical rows [v0, v0+V) as float32[V, dim] (written into `out` if given)."""
    if out is None:
        out = np.empty((V, dim), dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.shape == (V, dim)
    lib().synth_features(v0, V, dim, _p(out))
    return out


def features_at(ids: np.ndarray, dim: int) -> np.ndarray:
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.empty((len(ids), dim), dtype=np.float32)
    lib().synth_features_at(_p(ids), len(ids), dim, _p(out))
    return out


def write_feature_file(path: str, V: int, dim: int, header_bytes: int = 4096, stride: int | None = None) -> int:
    """Writes the canonical feature file; returns the row stride (roundup(4*dim, 512))."""
    if stride is None:
        stride = (4 * dim + 511) // 512 * 512
    rc = lib().synth_write_feature_file(path.encode(), V, dim, header_bytes, stride)
    if rc != 0:
        raise OSError(f"synth_write_feature_file({path}) -> {rc}")
    return stride


def train_set(V: int, seed: int = HELIOS_SEED, pct: int = 1) -> np.ndarray:
    L = lib()
    n = L.synth_train_set(V, seed, pct, None)
    out = np.empty(n, dtype=np.int64)
    L.synth_train_set(V, seed, pct, _p(out))
    return out


def epoch_batches(train: np.ndarray, B: int, epoch: int, seed: int = HELIOS_SEED, drop_last: bool = False) -> list[np.ndarray]:
    train = np.ascontiguousarray(train, dtype=np.int64)
    order = np.empty_like(train)
    lib().synth_epoch_order(_p(train), len(train), seed, epoch, _p(order))
    out = [order[i:i + B] for i in range(0, len(order), B)]
    if drop_last and out and len(out[-1]) < B:
        out.pop()
    return out


def batch_key(global_seed: int, epoch: int, b: int) -> int:
    return int(lib().synth_batch_key(global_seed & 0xFFFFFFFFFFFFFFFF, epoch, b))


def presample_key(global_seed: int, b: int) -> int:
    return batch_key(~global_seed & 0xFFFFFFFFFFFFFFFF, 0, b)
