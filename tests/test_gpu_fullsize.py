"""GPU parity at BASELINE.json sizes in the launch configuration bench.py times (execution plan,
CUDA graphs, 8 batches in flight, ticketed host rows), against the CPU oracle, bit-exact:

* C2 (ogbn-products-shaped, 2.4 M / 62 M, dim 100, fully HBM-cached): the first 20 batches of the
  epoch, every output (nodes, per-hop block CSR, feature bytes, per-tier counts).
* C3 (ogbn-papers100M-shaped) at s = 0.1 (11.1 M / 160 M, dim 128, HBM 10 % + pinned host 90 %,
  host tier packed in hot-rank order): the first 16 batches, same checks; and C3 at full size
  (111 M / 1.6 B): the first 8 batches (also checked on every bench.py run, `parity` in its JSON).
* Cross-slot isolation: batches replayed through different slots in a different order give the
  same bytes.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import workloads  # noqa: E402


def setup(H, cfg, flags=0):
    inp = workloads.make_inputs(cfg, table=True)
    g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices)
    hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
    pk = workloads.presample_keys(len(inp.batches))
    for b in range(len(inp.batches)):
        H.helios_presample(g, torch.as_tensor(inp.batches[b]).cuda(), cfg.B, cfg.fanouts, [pk[b]], hot)
    H.helios_graph_sync(g)
    Hr, S = workloads.tier_rows(cfg)
    if cfg.hbm_frac + cfg.host_frac >= 1.0:
        S = max(0, cfg.V - Hr)
    # staged caches as the bench builds them: 14 stagers, last 60 % of each batch's host chunks reserved
    skw = dict(stage_workers=14, stage_reserve=0.6) if flags & H.HOST_STAGED else {}
    c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=inp.table, flags=flags, **skw)
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, Hr, S)
    return inp, g, c, dref


def check_batches(H, inp, g, c, dref, n_batches, depth=8, order=None, group=1):
    cfg = inp.cfg
    keys = workloads.batch_keys(0, len(inp.batches))
    full = [b for b in range(len(inp.batches)) if len(inp.batches[b]) == cfg.B][:n_batches]
    if order == "reversed":
        full = full[::-1]
    p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=depth, group=group)
    stream = torch.cuda.current_stream()
    seeds = {b: torch.as_tensor(inp.batches[b]).cuda() for b in full}
    got = {}
    for start in range(0, len(full), p.positions):
        idx = full[start:start + p.positions]
        for k, b in enumerate(idx):
            H.helios_plan_submit(p, k, seeds[b], keys[b], stream)
        for k, b in enumerate(idx):
            H.helios_plan_wait(p, k, stream)
        H.helios_sync(c)
        for k, b in enumerate(idx):
            blocks, feats, stats = p.outputs[k]
            out = blocks.to_host()
            n = len(out["nodes"])
            got[b] = (out, feats[:n].cpu().numpy(), stats.cpu().numpy())
    p.free()
    for b in full:
        out, feats, stats = got[b]
        orc = oracle.sample(inp.graph.indptr, inp.graph.indices, inp.batches[b], cfg.fanouts, keys[b])
        assert np.array_equal(out["nodes"], orc.nodes), f"batch {b}: nodes"
        for h in range(len(cfg.fanouts)):
            assert np.array_equal(out["block_indptr"][h], orc.block_indptr[h]), f"batch {b}: hop {h} indptr"
            assert np.array_equal(out["block_indices"][h], orc.block_indices[h]), f"batch {b}: hop {h} indices"
        assert np.array_equal(feats, oracle.gather(orc.nodes, cfg.R, table=inp.table)), f"batch {b}: features"
        assert stats.tolist() == oracle.lookup_counts(dref, orc.nodes).tolist(), f"batch {b}: tier counts"
    return got


@pytest.fixture(scope="module")
def H():
    from paper_2310_00837_b200 import helios
    return helios


def test_c2_full_size_plan(H, monkeypatch):
    inp, g, c, dref = setup(H, workloads.CONFIGS["C2"])
    a = check_batches(H, inp, g, c, dref, 20)
    # the same batches through other slots, reversed: identical bytes (no state leaks across slots)
    b = check_batches(H, inp, g, c, dref, 20, depth=5, order="reversed")
    for k in a:
        assert np.array_equal(a[k][1], b[k][1])
    # and through plan groups of 4 (one launch of each kernel for 4 batches)
    b = check_batches(H, inp, g, c, dref, 20, depth=3, group=4)
    for k in a:
        assert np.array_equal(a[k][1], b[k][1])
    # and with the shared-memory tile dedup (HELIOS_SAMPLE_DEDUP=smem, read at plan creation)
    monkeypatch.setenv("HELIOS_SAMPLE_DEDUP", "smem")
    b = check_batches(H, inp, g, c, dref, 20, depth=12)
    for k in a:
        assert np.array_equal(a[k][1], b[k][1])
    monkeypatch.delenv("HELIOS_SAMPLE_DEDUP")
    # and with the other fused-gather variants (read at cache build): 8 loads per lane, a cp.async
    # shared-memory ring
    for env in ({"HELIOS_GATHER_VU": "8"}, {"HELIOS_GATHER_ASYNC": "4"}):
        for k in ("HELIOS_GATHER_VU", "HELIOS_GATHER_ASYNC"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        hot = torch.zeros(inp.cfg.V, dtype=torch.int64, device="cuda")
        c2 = H.helios_cache_build(g, hot, inp.cfg.R, inp.cfg.V, 0, host_table=inp.table)
        d2, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, inp.cfg.V, 0)
        b = check_batches(H, inp, g, c2, d2, 20, depth=12)
        for k in a:
            assert np.array_equal(a[k][1], b[k][1])
        c2.free()
    c.free()
    g.free()


@pytest.mark.parametrize("staged", [False, True])
def test_c3_scaled_plan(H, staged):
    cfg = workloads.scaled(workloads.CONFIGS["C3"], 0.1)
    inp, g, c, dref = setup(H, cfg, flags=H.HOST_STAGED if staged else 0)
    got = check_batches(H, inp, g, c, dref, 16)
    assert sum(int(v[2][2]) for v in got.values()) > 0   # host-tier rows were exercised
    c.free()
    g.free()


def test_c3_full_size_plan(H):
    """C3 at BASELINE.json's full size (111 M / 1.6 B, 56.8 GB feature table, 51 GB packed host tier):
    8 batches through the bench's plan configuration (dynamic staged host tier, 12 in flight), every
    output bit-exact."""
    cfg = workloads.CONFIGS["C3"]
    import os
    avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    if avail < 150e9:
        pytest.skip(f"needs ~125 GB of host RAM for the table + packed host tier, {avail / 1e9:.0f} GB available")
    inp, g, c, dref = setup(H, cfg, flags=H.HOST_STAGED)
    got = check_batches(H, inp, g, c, dref, 24, depth=12)
    got2 = check_batches(H, inp, g, c, dref, 16, depth=4, group=4)   # plan groups (bench --group)
    for k in got2:
        assert np.array_equal(got[k][1], got2[k][1])
    assert sum(int(v[2][2]) for v in got.values()) > 0
    c.free()
    g.free()
