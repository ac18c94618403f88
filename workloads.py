"""Workload configurations (BASELINE.json configs / SURVEY.md §8(d)) and setup glue shared by
tests/, bench.py and __graft_entry__.smoke().

A Workload owns the synthetic inputs (graph, canonical feature table and/or feature file, train
set, batches, keys) and, on a GPU, the library handles (graph, hotness, cache).  Inputs come only
from `synth`; nothing here computes any step of the method.
"""
from __future__ import annotations

import math
import os
import tempfile
import time
from dataclasses import dataclass, field

import numpy as np

import synth

SEED = synth.HELIOS_SEED


@dataclass
class Config:
    name: str
    V: int
    E: int
    dim: int
    B: int
    fanouts: list
    hbm_frac: float        # fraction of V in the HBM tier (per GPU for the sweep config)
    host_frac: float       # fraction of V in the host tier
    train_pct: int = 1     # 1% training vertices
    note: str = ""

    @property
    def R(self) -> int:
        return 4 * self.dim


CONFIGS = {
    # configs[0]: tiny, every tier (file tier = rest)
    "C1": Config("C1", 10_000, 200_000, 128, 256, [10, 5], 0.10, 0.40, train_pct=100,
                 note="synthetic power-law 10k/200k, dim 128, fanout [10,5], batch 256, HBM 10%/host 40%/file rest"),
    # configs[1]: ogbn-products-shaped, in-memory regime
    "C2": Config("C2", 2_400_000, 62_000_000, 100, 1024, [15, 10, 5], 1.0, 0.0,
                 note="ogbn-products-shaped 2.4M/62M, dim 100, fanout [15,10,5], batch 1024, fully HBM-cached"),
    # configs[2]: ogbn-papers100M-shaped, HBM + pinned host
    "C3": Config("C3", 111_000_000, 1_600_000_000, 128, 1024, [15, 10, 5], 0.10, 0.90,
                 note="ogbn-papers100M-shaped 111M/1.6B, dim 128, fanout [15,10,5], batch 1024, HBM 10% + pinned host 90%"),
    # configs[3]: IGB-large-shaped, HBM + host + file (scaled by s to fit the box, reported)
    "C4": Config("C4", 100_000_000, 1_200_000_000, 1024, 1024, [15, 10, 5], 0.10, 0.40,
                 note="IGB-large-shaped 100M/1.2B, dim 1024, HBM 10%/host 40%/file rest"),
}


def scaled(cfg: Config, s: float) -> Config:
    """Capacity scaling rule: V and E by s; degree, skew, dim, B, f, tier % kept."""
    if s == 1.0:
        return cfg
    c = Config(**{**cfg.__dict__})
    c.V = max(1000, int(cfg.V * s))
    c.E = max(1000, int(cfg.E * s))
    c.name = f"{cfg.name}@s={s:g}"
    return c


@dataclass
class Inputs:
    cfg: Config
    graph: synth.Graph
    table: np.ndarray | None          # canonical rows [V, dim] fp32 (host)
    feature_path: str | None
    header: int
    stride: int
    train: np.ndarray
    batches: list
    gen_s: float = 0.0
    extra: dict = field(default_factory=dict)


def make_inputs(cfg: Config, table: bool = True, file: bool = False, workdir: str | None = None,
                epoch: int = 0, table_buffer=None) -> Inputs:
    t0 = time.time()
    g = synth.graph(cfg.V, cfg.E, seed=SEED)
    tab = None
    if table:
        tab = table_buffer if table_buffer is not None else np.empty((cfg.V, cfg.dim), dtype=np.float32)
        synth.features(cfg.V, cfg.dim, out=tab)
    path, header, stride = None, 4096, (cfg.R + 511) // 512 * 512
    if file:
        d = workdir or tempfile.mkdtemp(prefix="helios_")
        path = os.path.join(d, f"features_{cfg.name}.bin")
        stride = synth.write_feature_file(path, cfg.V, cfg.dim, header_bytes=header)
    train = synth.train_set(cfg.V, SEED, cfg.train_pct)
    batches = synth.epoch_batches(train, cfg.B, epoch, SEED)
    return Inputs(cfg, g, tab, path, header, stride, train, batches, gen_s=time.time() - t0)


def tier_rows(cfg: Config, world_size: int = 1) -> tuple[int, int]:
    """(H per GPU, S) rows for the config's tier fractions."""
    H = int(round(cfg.hbm_frac * cfg.V))
    if cfg.hbm_frac >= 1.0:
        H = math.ceil(cfg.V / world_size)
    S = int(round(cfg.host_frac * cfg.V))
    return H, S


def presample_keys(n: int) -> list[int]:
    return [synth.presample_key(SEED, b) for b in range(n)]


def batch_keys(epoch: int, n: int) -> list[int]:
    return [synth.batch_key(SEED, epoch, b) for b in range(n)]
