"""CPU checks of bench.py: the --impl reference arm (the oracle on host cores) prints one JSON line
with the driver contract's keys, and the capacity/tier helpers behave."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_contract():
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config",
                                   "C1", "--steps", "3", "--warmup", "1"], cwd=ROOT, text=True, timeout=300)
    lines = [l for l in out.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 3 and d["warmup"] == 1 and d["value"] > 0
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["vs_baseline"] is None
    assert d["config"]["workload"] == "C1"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_capacity_and_tier_helpers():
    sys.path.insert(0, ROOT)
    import bench
    import workloads
    C = workloads.CONFIGS
    assert not bench.has_file_tier(C["C2"]) and not bench.has_file_tier(C["C3"])
    assert bench.has_file_tier(C["C1"]) and bench.has_file_tier(C["C4"])
    assert bench.keeps_table(C["C1"]) and bench.keeps_table(C["C3"]) and not bench.keeps_table(C["C4"])
    assert bench.pick_scale(C["C1"], 1) == 1.0
    huge = workloads.Config("huge", 10**12, 10**13, 1024, 1024, [15], 0.1, 0.4)
    s = bench.pick_scale(huge, 1)
    assert 0.01 <= s < 1.0
    sc = workloads.scaled(C["C4"], 0.1)
    assert sc.V == C["C4"].V // 10 and sc.dim == 1024 and sc.fanouts == C["C4"].fanouts
    H, S = workloads.tier_rows(C["C3"])
    assert H == 11_100_000 and S == 99_900_000
    H2, _ = workloads.tier_rows(C["C2"], world_size=3)
    assert H2 * 3 >= C["C2"].V


def test_interval_union():
    """The busy time of overlapping launches (roofline denominator) against brute force on a grid."""
    sys.path.insert(0, ROOT)
    import random

    import bench
    assert bench.interval_union([]) == 0.0
    assert bench.interval_union([(0, 1), (2, 3)]) == 2.0
    assert bench.interval_union([(0, 2), (1, 3), (5, 6), (5.5, 5.7)]) == 4.0
    rng = random.Random(5)
    for _ in range(50):
        iv = []
        for _ in range(rng.randint(1, 12)):
            a = rng.randint(0, 40)
            iv.append((a, a + rng.randint(0, 10)))
        covered = sum(1 for t in range(60) if any(a <= t < b for a, b in iv))
        assert bench.interval_union(iv) == covered


def test_sampling_sector_count():
    """bench.sampling_accesses: exact on full rows; the k < d expectation matches a Monte-Carlo draw."""
    sys.path.insert(0, ROOT)
    import numpy as np

    import bench
    # one hop, rows: v0 d=3 (k=d, one sector), v1 d=20 starting at 3 (k=d: sectors 0..2), v2 d=400, f=5
    indptr = np.array([0, 3, 23, 423], dtype=np.int64)
    batch = {"nodes": np.array([0, 1, 2]), "level_counts": np.array([3, 3])}
    got = bench.sampling_accesses(batch, indptr, [5])
    # v0: k=3=d -> span 1; v1: k=5<d=20 -> expectation; v2: k=5<400 -> expectation
    rng = np.random.default_rng(0)
    mc = 0.0
    for base, d in ((3, 20), (23, 400)):
        t = 0
        for _ in range(4000):
            pos = base + rng.choice(d, 5, replace=False)
            t += len(np.unique(pos // 8))
        mc += t / 4000
    expect_sectors = 3 + 1 + mc + 3          # indptr per row + v0's sector + sampled + directory
    assert abs(got["sectors"] - expect_sectors) < 0.25
    assert got["stream_bytes"] == 4 * (3 + 5 + 5) + 4 * 4 + 8 * 3


def test_oracle_baseline_threads():
    """The P-core leg of cpu_baseline: several threads each prepare independent batches; every batch
    equals the single-threaded oracle's (the threads share no state but the batch counter)."""
    import bench
    import oracle
    import workloads
    cfg = workloads.Config("tiny", 3000, 30_000, 16, 64, [5, 3], 0.1, 0.4, train_pct=100)
    inp = workloads.make_inputs(cfg, table=True)
    keys = workloads.batch_keys(0, len(inp.batches))
    seen = {}

    def check(b, ob, feats):
        seen[b] = (ob.nodes.copy(), feats.copy())

    r = bench.run_oracle_baseline(inp, keys, 5.0, check=check, threads=3)
    assert r["threads"] == 3 and r["batches"] == len(seen) > 0 and r["value"] > 0
    for b, (nodes, feats) in list(seen.items())[:5]:
        ob = oracle.sample(inp.graph.indptr, inp.graph.indices, inp.batches[b], cfg.fanouts, keys[b])
        assert np.array_equal(nodes, ob.nodes)
        assert np.array_equal(feats, oracle.gather(ob.nodes, cfg.R, table=inp.table))
    assert bench.cpu_model()
