"""GPU parity of the execution plan (helios_plan_*): CUDA-graph replay and direct launches, 1-3
in-flight slots, device and host seeds, all three tiers (C1 incl. the IO rings) and the HBM+host
config shape (medium graph) — every batch bit-exact against the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402
import workloads  # noqa: E402


@pytest.fixture(scope="module")
def H():
    from paper_2310_00837_b200 import helios
    return helios


@pytest.fixture(scope="module")
def c1(tmp_path_factory):
    return workloads.make_inputs(workloads.CONFIGS["C1"], table=True, file=True,
                                 workdir=str(tmp_path_factory.mktemp("c1p")))


def build(H, inp, Hr, S, flags=0):
    # staged-mode caches use 3 stager threads, stage at most 70 % of each batch's host rows and reserve
    # the last 50 % for the stagers
    cfg = inp.cfg
    g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices)
    hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
    pk = workloads.presample_keys(len(inp.batches))
    H.helios_presample(g, torch.as_tensor(np.concatenate(inp.batches)).cuda(), cfg.B, cfg.fanouts, pk, hot)
    c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=inp.table, feature_path=inp.feature_path,
                             header_bytes=inp.header, file_stride=inp.stride, flags=flags, stage_workers=3,
                             stage_frac=0.7, stage_reserve=0.5)
    return g, hot, c


def check_slot(p, slot, inp, seeds, key, dref):
    cfg = inp.cfg
    blocks, feats, stats = p.outputs[slot]
    got = blocks.to_host()
    orc = oracle.sample(inp.graph.indptr, inp.graph.indices, seeds, cfg.fanouts, key)
    assert np.array_equal(got["nodes"], orc.nodes)
    for h in range(len(cfg.fanouts)):
        assert np.array_equal(got["block_indptr"][h], orc.block_indptr[h])
        assert np.array_equal(got["block_indices"][h], orc.block_indices[h])
    if feats is not None:
        n = len(orc.nodes)
        assert np.array_equal(feats[:n].cpu().numpy(), oracle.gather(orc.nodes, cfg.R, table=inp.table))
        assert stats.cpu().tolist() == oracle.lookup_counts(dref, orc.nodes).tolist()


@pytest.mark.parametrize("depth,flags,host_seeds,staged", [(2, 0, False, False), (1, 0, True, False),
                                                          (3, 0, False, False), (2, 1, True, False),
                                                          (3, 0, False, True), (1, 1, True, True),
                                                          (1, 4, False, False), (3, 4, True, False),
                                                          (2, 4, False, True), (2, 2, False, False),
                                                          (3, 8, False, False), (2, 8, True, True),
                                                          (6, 0, False, False), (6, 1, False, True),
                                                          (6, 8, False, False), (4, 9, True, False)])
def test_plan_c1_epoch(H, c1, depth, flags, host_seeds, staged):
    cfg = c1.cfg
    Hr, S = workloads.tier_rows(cfg)
    g, hot, c = build(H, c1, Hr, S, flags=H.HOST_ALIAS | (H.HOST_STAGED if staged else 0))
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, Hr, S, host_slot_is_id=True)
    p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=depth, flags=flags)
    keys = workloads.batch_keys(0, len(c1.batches))
    stream = torch.cuda.current_stream()
    nb = len(c1.batches)
    for start in range(0, nb, depth):
        idx = list(range(start, min(nb, start + depth)))
        live = []   # device seeds must stay allocated until their batch completes (helios.h)
        for k, b in enumerate(idx):
            seeds = c1.batches[b] if host_seeds else torch.as_tensor(c1.batches[b]).cuda()
            live.append(seeds)
            H.helios_plan_submit(p, k, seeds, keys[b], stream, timing=(b % 2 == 0))
        for k, b in enumerate(idx):
            H.helios_plan_wait(p, k, stream)
        H.helios_sync(c)
        for k, b in enumerate(idx):
            check_slot(p, k, c1, c1.batches[b], keys[b], dref)
        if depth > 1 or start % 2 == 0:
            t = H.helios_plan_timing(p, 0)
            assert t.sample_ms > 0 and t.gather_ms > 0
            assert (t.link_ms > 0) == p.link
            assert t.t_start == -1.0   # never marked
    p.free()
    c.free()


@pytest.mark.parametrize("depth,group,flags,host_seeds,staged,partial",
                         [(2, 2, 0, False, False, False), (2, 4, 0, True, False, False), (3, 3, 1, False, False, False),
                          (2, 4, 0, False, True, False), (1, 4, 2, True, False, False), (2, 3, 0, False, False, True),
                          (1, 2, 1, True, True, True)])
def test_plan_groups_c1_epoch(H, c1, depth, group, flags, host_seeds, staged, partial):
    """Plan groups (desc.group): each kernel of a slot's chain launched once for `group` batches
    (gridDim.y).  Every batch of the C1 epoch, at every position, equals the oracle (sampling, three-
    tier gather incl. the IO rings, tier counts); per-position readback; partial groups launched by
    helios_plan_wait (partial=True: only some positions of a group are submitted, the others run as
    empty batches and keep nothing of their previous batch visible through readback)."""
    cfg = c1.cfg
    Hr, S = workloads.tier_rows(cfg)
    g, hot, c = build(H, c1, Hr, S, flags=H.HOST_ALIAS | (H.HOST_STAGED if staged else 0))
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, Hr, S, host_slot_is_id=True)
    p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=depth, flags=flags, group=group)
    assert p.positions == depth * group
    keys = workloads.batch_keys(0, len(c1.batches))
    stream = torch.cuda.current_stream()
    nb = len(c1.batches)
    P = p.positions
    rnd = 0
    for start in range(0, nb, P):
        idx = list(range(start, min(nb, start + P)))
        if partial and rnd % 2 == 1:
            idx = idx[: max(1, group - 1)]   # the first group is left incomplete
        rnd += 1
        live = []
        for k, b in enumerate(idx):
            seeds = c1.batches[b] if host_seeds else torch.as_tensor(c1.batches[b]).cuda()
            live.append(seeds)
            H.helios_plan_submit(p, k, seeds, keys[b], stream, timing=(b % 2 == 0), readback=True)
        for k, b in enumerate(idx):
            H.helios_plan_wait(p, k, stream)
        H.helios_sync(c)
        for k, b in enumerate(idx):
            check_slot(p, k, c1, c1.batches[b], keys[b], dref)
            rb = H.helios_plan_readback(p, k)
            orc_n = p.outputs[k][0].level_counts.cpu().numpy()
            assert rb[: len(cfg.fanouts) + 1].tolist() == orc_n.tolist()
            assert rb[len(cfg.fanouts) + 1:].tolist() == p.outputs[k][2].cpu().tolist()
        if partial and len(idx) < group:   # positions of the group not submitted ran as empty batches
            for k in range(len(idx), group):
                assert int(p.outputs[k][0].level_counts[0].item()) == 0
    with pytest.raises(H.HeliosError) as e:
        H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=2, group=5)
    assert e.value.name == "E_INVALID"
    p.free()
    c.free()


def test_plan_sample_only_medium(H):
    gr = synth.graph(400_000, 8_000_000, seed=33)
    g = H.helios_graph_load(gr.indptr, gr.indices)
    fan = [15, 10, 5]
    p = H.helios_plan_create(g, None, 1024, fan, depth=2)
    rng = np.random.default_rng(4)
    inp = workloads.Inputs(workloads.Config("m", gr.V, gr.E, 1, 1024, fan, 0, 0), gr, None, None, 0, 0, None, [])
    for it in range(3):
        seeds = [rng.choice(gr.V, 1024 - 100 * k, replace=False) for k in range(2)]
        keys = [it * 7 + 1, it * 7 + 2]
        dev = [torch.as_tensor(x).cuda() for x in seeds]   # alive until the batches complete
        for k in range(2):
            H.helios_plan_submit(p, k, dev[k], keys[k])
        torch.cuda.synchronize()
        for k in range(2):
            H.helios_plan_wait(p, k)
            H.helios_graph_sync(g)
            check_slot(p, k, inp, seeds[k], keys[k], None)
    with pytest.raises(H.HeliosError) as e:
        H.helios_plan_submit(p, 0, torch.arange(2000, device="cuda"), 1)
    assert e.value.name == "E_CAPACITY"
    p.free()


def test_staged_stress_many_batches(H):
    """Staged host tier under sustained load: 4000 batches through a 6-slot plan (a few hundred
    thousand chunk hand-offs between GPU stage warps and host stager threads) must finish without the
    watchdog firing, and the final batches must stay bit-exact."""
    cfg = workloads.Config("stress", 200_000, 3_000_000, 64, 1024, [15, 10, 5], 0.05, 0.95, train_pct=100)
    inp = workloads.make_inputs(cfg, table=True)
    Hr, S = int(0.05 * cfg.V), cfg.V - int(0.05 * cfg.V)
    g, hot, c = build(H, inp, Hr, S, flags=H.HOST_STAGED)
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, Hr, S)
    p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=6)
    keys = workloads.batch_keys(0, len(inp.batches))
    seeds = [torch.as_tensor(b).cuda() for b in inp.batches[:64]]
    n = 4000
    for i in range(n):
        H.helios_plan_submit(p, i % 6, seeds[i % 64], keys[i % 64])
    for k in range(6):
        H.helios_plan_wait(p, k)
    H.helios_sync(c)
    for k in range(6):
        b = (n - 6 + k) % 64
        check_slot(p, (n - 6 + k) % 6, inp, inp.batches[b], keys[b], dref)
    assert c.info().host_rows == S
    p.free()
    c.free()


def test_plan_readback(H, c1):
    """HELIOS_SUBMIT_READBACK / helios_plan_readback: the host copy equals the slot's device level
    counts and tier stats (= the oracle's); E_STATE for a batch submitted without it."""
    cfg = c1.cfg
    Hr, S = workloads.tier_rows(cfg)
    g, hot, c = build(H, c1, Hr, S)
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, Hr, S)
    p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=3)
    keys = workloads.batch_keys(0, len(c1.batches))
    for b in range(6):
        k = b % 3
        if b >= 3:
            got = H.helios_plan_readback(p, k)
            ob = oracle.sample(c1.graph.indptr, c1.graph.indices, c1.batches[b - 3], cfg.fanouts, keys[b - 3])
            assert got[: len(cfg.fanouts) + 1].tolist() == ob.level_counts.tolist()
            assert got[len(cfg.fanouts) + 1:].tolist() == oracle.lookup_counts(dref, ob.nodes).tolist()
        H.helios_plan_submit(p, k, c1.batches[b], keys[b], readback=True)
    H.helios_plan_submit(p, 0, c1.batches[0], keys[0])
    with pytest.raises(H.HeliosError) as e:
        H.helios_plan_readback(p, 0)
    assert e.value.name == "E_STATE"
    H.helios_sync(c)
    p.free()
    c.free()


def test_plan_timing_marked(H, c1):
    """helios_plan_mark + HELIOS_SUBMIT_TIMING: per-batch offsets are ordered (start <= end of sampling
    <= end) and consistent with the durations; batches of different slots share the origin."""
    cfg = c1.cfg
    Hr, S = workloads.tier_rows(cfg)
    g, hot, c = build(H, c1, Hr, S)
    p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=2)
    keys = workloads.batch_keys(0, len(c1.batches))
    stream = torch.cuda.current_stream()
    H.helios_plan_mark(p, stream)
    for b in range(4):
        H.helios_plan_submit(p, b % 2, c1.batches[b], keys[b], stream, timing=True)
    for k in range(2):
        H.helios_plan_wait(p, k, stream)
    H.helios_sync(c)
    ends = []
    for k in range(2):
        for back in range(2):
            t = H.helios_plan_timing(p, k, back)
            assert 0 <= t.t_start <= t.t_gather <= t.t_end
            assert abs((t.t_gather - t.t_start) - t.sample_ms) < 1e-2
            assert abs((t.t_end - t.t_gather) - t.gather_ms) < 1e-2
            ends.append(t.t_end)
    assert max(ends) < 10_000
    with pytest.raises(H.HeliosError) as e:
        H.helios_plan_timing(p, 0, 2)
    assert e.value.name == "E_RANGE"
    p.free()
    c.free()


TRACE_CHECK = r"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle, workloads
from paper_2310_00837_b200 import helios as H
assert H.SO_PATH.endswith("libhelios_trace.so")
c1 = workloads.make_inputs(workloads.CONFIGS["C1"], table=True)
cfg = c1.cfg
Hr, _ = workloads.tier_rows(cfg)
S = cfg.V - Hr   # HBM + host tiers only (no feature file in this check)
g = H.helios_graph_load(c1.graph.indptr, c1.graph.indices)
hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
H.helios_presample(g, torch.as_tensor(np.concatenate(c1.batches)).cuda(), cfg.B, cfg.fanouts,
                   workloads.presample_keys(len(c1.batches)), hot)
c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=c1.table, flags=H.HOST_ALIAS)
p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=3, flags=H.PLAN_TRACE)
keys = workloads.batch_keys(0, len(c1.batches))
for b in range(6):
    H.helios_plan_submit(p, b % 3, c1.batches[b], keys[b])
    if b % 3 == 2:
        for k in range(3):
            H.helios_plan_wait(p, k)
        H.helios_sync(c)
        for k in range(3):
            ob = oracle.sample(c1.graph.indptr, c1.graph.indices, c1.batches[b - 2 + k], cfg.fanouts, keys[b - 2 + k])
            blocks, feats, _ = p.outputs[k]
            assert np.array_equal(blocks.to_host()["nodes"], ob.nodes)
            assert np.array_equal(feats[: len(ob.nodes)].cpu().numpy(), oracle.gather(ob.nodes, cfg.R, table=c1.table))
for k in range(3):
    for back in range(2):
        t = H.helios_plan_trace(p, k, back).astype(np.int64)
        assert t.shape == (3 * len(cfg.fanouts) + 4, 2)
        assert (t[:, 0] > 0).all() and (t[:, 1] >= t[:, 0]).all()
        assert (t[1:, 0] >= t[:-1, 1] - 2000).all()   # each kernel starts after its predecessor ended (ns)
try:
    H.helios_plan_trace(p, 0, 2)
    raise SystemExit("expected E_RANGE")
except H.HeliosError as e:
    assert e.name == "E_RANGE"
print("trace ok")
"""


def test_plan_trace(H, c1):
    """HELIOS_PLAN_TRACE: E_INVALID in the product build; in the traced build (HELIOS_LIB=trace, run
    in a subprocess) outputs stay bit-exact, every kernel position of a batch ran, and each kernel of
    the chain starts after its predecessor ended (programmatic-dependency wait / stream order)."""
    import os
    import subprocess
    import sys
    cfg = c1.cfg
    Hr, S = workloads.tier_rows(cfg)
    g, hot, c = build(H, c1, Hr, S, flags=H.HOST_ALIAS)
    with pytest.raises(H.HeliosError) as e:
        H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=1, flags=H.PLAN_TRACE)
    assert e.value.name == "E_INVALID"
    c.free()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2310_00837_b200 import build as hb
    hb.build()   # both libraries; a no-op when they are up to date
    out = subprocess.run([sys.executable, "-c", TRACE_CHECK], cwd=root, env={**os.environ, "HELIOS_LIB": "trace"},
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "trace ok" in out.stdout, out.stderr[-3000:]
