"""GPU parity of helios_cache_build / helios_gather / helios_batch_prepare against the oracle.

* Directory: bit-exact vs oracle.cache_dir for several (world_size, rank, H, S, alias) cases.
* Gather: output bytes == oracle.gather (canonical rows) for every row, all three tiers (HBM,
  pinned host zero-copy, file through the GPU-initiated IO rings), row sizes 400/512/4096 B;
  per-tier row counts == oracle.lookup_counts.
* batch_prepare over the C1 epoch (every batch) == oracle sample + gather.
* IO rings: ring_depth 2 (wrap-around + back-pressure), fault injection -> latched E_IO.
"""
import os

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
                                 workdir=str(tmp_path_factory.mktemp("c1")))


@pytest.fixture(scope="module")
def c1_hot(H, c1):
    g = H.helios_graph_load(c1.graph.indptr, c1.graph.indices)
    keys = workloads.presample_keys(len(c1.batches))
    hot = torch.zeros(c1.cfg.V, dtype=torch.int64, device="cuda")
    H.helios_presample(g, torch.as_tensor(np.concatenate(c1.batches)).cuda(), c1.cfg.B, c1.cfg.fanouts, keys, hot)
    H.helios_graph_sync(g)
    return g, hot


@pytest.mark.parametrize("G,rank,Hr,S,alias", [(1, 0, 1000, 4000, False), (1, 0, 1000, 4000, True), (3, 2, 700, 500, False),
                                               (4, 1, 0, 9000, True), (1, 0, 20000, 0, False)])
def test_directory_parity(H, c1, c1_hot, G, rank, Hr, S, alias):
    g, hot = c1_hot
    c = H.helios_cache_build(g, hot, c1.cfg.R, Hr, S, host_table=c1.table, feature_path=c1.feature_path,
                             header_bytes=c1.header, file_stride=c1.stride, world_size=G, rank=rank,
                             flags=H.HOST_ALIAS if alias else 0)
    inf = c.info()
    dgpu = H.device_view(inf.dir, c1.cfg.V, torch.int64).cpu().numpy()
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), G, Hr, S, host_slot_is_id=alias)
    assert np.array_equal(dgpu, dref)
    c.free()


def gather_and_check(H, c, inp, nodes_np, stats_ref):
    R = inp.cfg.R
    nodes = torch.as_tensor(nodes_np).cuda()
    n = torch.tensor([len(nodes_np)], dtype=torch.int64, device="cuda")
    out = torch.full((max(1, len(nodes_np)), R), 0xAB, dtype=torch.uint8, device="cuda")
    stats = H.new_stats()
    H.helios_gather(c, nodes, n, out, stats)
    H.helios_sync(c)
    ref = oracle.gather(nodes_np, R, table=inp.table)
    assert np.array_equal(out[: len(nodes_np)].cpu().numpy(), ref)
    assert stats.cpu().numpy().tolist() == stats_ref.tolist()


@pytest.mark.parametrize("alias,staged,frac,reserve", [(False, False, 0, 0), (True, False, 0, 0), (False, True, 0.5, 0),
                                                       (True, True, 0.5, 0), (False, True, 1.0, 0), (False, True, 1.0, 0.6),
                                                       (True, True, 0.7, 0.7)])
def test_gather_three_tiers_c1(H, c1, c1_hot, alias, staged, frac, reserve):
    g, hot = c1_hot
    cfg = c1.cfg
    Hr, S = workloads.tier_rows(cfg)
    c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=c1.table, feature_path=c1.feature_path,
                             header_bytes=c1.header, file_stride=c1.stride,
                             flags=(H.HOST_ALIAS if alias else 0) | (H.HOST_STAGED if staged else 0),
                             stage_workers=3, stage_frac=frac, stage_reserve=reserve)
    assert c.info().file_rows == cfg.V - Hr - S
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, Hr, S, host_slot_is_id=alias)
    rng = np.random.default_rng(0)
    for n in (1, 31, 1000, 4097, cfg.V) + ((cfg.V,) * 6 if staged else ()):   # staged: GPU/CPU meeting points vary
        nodes = rng.permutation(cfg.V)[:n]
        gather_and_check(H, c, c1, nodes, oracle.lookup_counts(dref, nodes))
    c.free()


@pytest.mark.parametrize("dim", [100, 1024])
def test_gather_row_sizes(H, tmp_path, dim):
    V = 6000
    gr = synth.graph(V, 50_000, seed=5)
    table = synth.features(V, dim)
    path = str(tmp_path / "f.bin")
    stride = synth.write_feature_file(path, V, dim, header_bytes=4096)
    g = H.helios_graph_load(gr.indptr, gr.indices)
    hot = torch.as_tensor(np.random.default_rng(dim).integers(0, 50, V)).cuda()
    c = H.helios_cache_build(g, hot, 4 * dim, 1000, 2000, host_table=None, feature_path=path, header_bytes=4096,
                             file_stride=stride, ring_depth=16, io_rings=3)
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, 1000, 2000)
    nodes = np.random.default_rng(1).permutation(V)[:3001]
    inp = workloads.Inputs(workloads.Config("x", V, 0, dim, 0, [], 0, 0), gr, table, path, 4096, stride, None, [])
    gather_and_check(H, c, inp, nodes, oracle.lookup_counts(dref, nodes))
    c.free()


@pytest.mark.parametrize("sync", [False, True])
def test_io_ring_wraparound_and_fault(H, c1, c1_hot, sync):
    g, hot = c1_hot
    cfg = c1.cfg
    sf = H.IO_SYNC if sync else 0
    c = H.helios_cache_build(g, hot, cfg.R, 0, 0, host_table=None, feature_path=c1.feature_path,
                             header_bytes=c1.header, file_stride=c1.stride, ring_depth=2, io_rings=2, io_ctas=2,
                             flags=sf)
    nodes = np.random.default_rng(9).permutation(cfg.V)[:3000]
    gather_and_check(H, c, c1, nodes, np.array([0, 0, 0, 3000]))
    gather_and_check(H, c, c1, nodes[::-1].copy(), np.array([0, 0, 0, 3000]))   # sequences continue across batches
    c.free()
    c = H.helios_cache_build(g, hot, cfg.R, 0, 0, host_table=None, feature_path=c1.feature_path,
                             header_bytes=c1.header, file_stride=c1.stride, ring_depth=8, io_rings=2,
                             flags=H.IO_FAULT_AT | sf, io_fault_at=17)
    out = torch.empty((3000, cfg.R), dtype=torch.uint8, device="cuda")
    H.helios_gather(c, torch.as_tensor(nodes).cuda(), torch.tensor([3000], device="cuda"), out)
    with pytest.raises(H.HeliosError) as e:
        H.helios_sync(c)
    assert e.value.name == "E_IO"
    c.free()


@pytest.mark.parametrize("direct,async_d,vu,evict", [("1", "0", "4", "0"), ("1", "0", "8", "0"), ("0", "0", "4", "0"),
                                                     ("1", "4", "4", "0"), ("1", "8", "4", "0"), ("1", "0", "4", "1")])
def test_hbm_only_direct_gather(H, c1, c1_hot, direct, async_d, vu, evict, monkeypatch):
    """Caches whose rows all live in HBM run the fused lookup + gather kernel (default) instead of K3 + K4
    (HELIOS_GATHER_DIRECT=0), with register-staged loads (VU per lane) or a D-stage cp.async shared-memory
    ring (HELIOS_GATHER_ASYNC=D), optionally with an evict-first L2 policy (HELIOS_GATHER_EVICT=1):
    same bytes, same tier counts, out-of-range ids latch E_RANGE."""
    monkeypatch.setenv("HELIOS_GATHER_DIRECT", direct)
    monkeypatch.setenv("HELIOS_GATHER_ASYNC", async_d)
    monkeypatch.setenv("HELIOS_GATHER_VU", vu)
    monkeypatch.setenv("HELIOS_GATHER_EVICT", evict)
    g, hot = c1_hot
    cfg = c1.cfg
    c = H.helios_cache_build(g, hot, cfg.R, cfg.V, 0, host_table=c1.table)
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, cfg.V, 0)
    rng = np.random.default_rng(11)
    for n in (1, 31, 257, 1000, cfg.V):
        nodes = rng.permutation(cfg.V)[:n]
        gather_and_check(H, c, c1, nodes, oracle.lookup_counts(dref, nodes))
    bad = torch.tensor([3, cfg.V + 5, 7], dtype=torch.int64, device="cuda")
    out = torch.empty((3, cfg.R), dtype=torch.uint8, device="cuda")
    H.helios_gather(c, bad, torch.tensor([3], device="cuda"), out)
    with pytest.raises(H.HeliosError) as e:
        H.helios_sync(c)
    assert e.value.name == "E_RANGE"
    c.free()


@pytest.mark.parametrize("split", ["1", "0"])
@pytest.mark.parametrize("staged,reserve", [(False, 0), (True, 0), (True, 0.7)])
def test_split_host_kernel(H, c1, c1_hot, staged, reserve, split, monkeypatch):
    """Host-tier rows in their own 64-thread kernel behind the HBM part (the default, split = 1) and in
    the combined kernel (HELIOS_GATHER_SPLIT_HOST=0, 2 host warps per 8), zero-copy, dynamic staged and
    reserved staged: three-tier gathers and a C1 plan stay bit-exact."""
    monkeypatch.setenv("HELIOS_GATHER_SPLIT_HOST", split)
    g, hot = c1_hot
    cfg = c1.cfg
    Hr, S = workloads.tier_rows(cfg)
    c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=c1.table, feature_path=c1.feature_path,
                             header_bytes=c1.header, file_stride=c1.stride,
                             flags=H.HOST_STAGED if staged else 0, stage_workers=3, stage_reserve=reserve)
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, Hr, S)
    rng = np.random.default_rng(5)
    for n in (1, 999, cfg.V, cfg.V):
        nodes = rng.permutation(cfg.V)[:n]
        gather_and_check(H, c, c1, nodes, oracle.lookup_counts(dref, nodes))
    p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=3)
    keys = workloads.batch_keys(0, len(c1.batches))
    live = [torch.as_tensor(b).cuda() for b in c1.batches[:9]]
    for i in range(9):
        H.helios_plan_submit(p, i % 3, live[i], keys[i])
        if i % 3 == 2:
            for k in range(3):
                H.helios_plan_wait(p, k)
            H.helios_sync(c)
            for k in range(3):
                b = i - 2 + k
                blocks, feats, stats = p.outputs[k]
                orc = oracle.sample(c1.graph.indptr, c1.graph.indices, c1.batches[b], cfg.fanouts, keys[b])
                assert np.array_equal(blocks.to_host()["nodes"], orc.nodes)
                assert np.array_equal(feats[: len(orc.nodes)].cpu().numpy(), oracle.gather(orc.nodes, cfg.R, table=c1.table))
                assert stats.cpu().tolist() == oracle.lookup_counts(dref, orc.nodes).tolist()
    p.free()
    c.free()


@pytest.mark.parametrize("io_sms,sync", [(8, False), (16, False), (48, True)])
def test_io_green_context(H, c1, c1_hot, io_sms, sync):
    """NEXT-3: the IO kernel confined to a green-context SM partition (the analog of the paper's MPS
    cap): three-tier gathers stay bit-exact, the provisioned SM count is
    reported, and a plan of C1 batches (sampling + gather on the primary context, IO on the partition)
    completes."""
    g, hot = c1_hot
    cfg = c1.cfg
    Hr, S = workloads.tier_rows(cfg)
    c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=c1.table, feature_path=c1.feature_path,
                             header_bytes=c1.header, file_stride=c1.stride, io_ctas=4, io_sms=io_sms,
                             flags=H.IO_SYNC if sync else 0)
    got = c.info().io_sms
    assert io_sms <= got < 148, got
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, Hr, S)
    rng = np.random.default_rng(io_sms)
    for n in (1, 1000, cfg.V):
        nodes = rng.permutation(cfg.V)[:n]
        gather_and_check(H, c, c1, nodes, oracle.lookup_counts(dref, nodes))
    reads0 = c.info().io_reads
    p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=3)
    keys = workloads.batch_keys(0, len(c1.batches))
    for i, b in enumerate(c1.batches[:12]):
        H.helios_plan_submit(p, i % 3, torch.as_tensor(b).cuda(), keys[i])
    for k in range(3):
        H.helios_plan_wait(p, k)
    H.helios_sync(c)
    assert c.info().io_reads > reads0
    p.free()
    c.free()


def test_batch_prepare_c1_epoch(H, c1, c1_hot):
    g, hot = c1_hot
    cfg = c1.cfg
    Hr, S = workloads.tier_rows(cfg)
    c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=c1.table, feature_path=c1.feature_path,
                             header_bytes=c1.header, file_stride=c1.stride, flags=H.HOST_ALIAS)
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, Hr, S, host_slot_is_id=True)
    blocks = H.Blocks.allocate(cfg.B, cfg.fanouts, g.V, g.E)
    feats = torch.empty((blocks.nodes.numel(), cfg.R), dtype=torch.uint8, device="cuda")
    stats = H.new_stats()
    keys = workloads.batch_keys(0, len(c1.batches))
    for seeds, key in zip(c1.batches, keys):
        H.helios_batch_prepare(g, c, torch.as_tensor(seeds).cuda(), cfg.fanouts, key, blocks, feats, stats)
        H.helios_sync(c)
        got = blocks.to_host()
        orc = oracle.sample(c1.graph.indptr, c1.graph.indices, seeds, cfg.fanouts, key)
        assert np.array_equal(got["nodes"], orc.nodes)
        for h in range(len(cfg.fanouts)):
            assert np.array_equal(got["block_indptr"][h], orc.block_indptr[h])
            assert np.array_equal(got["block_indices"][h], orc.block_indices[h])
        n = len(orc.nodes)
        ref = oracle.gather(orc.nodes, cfg.R, table=c1.table)
        assert np.array_equal(feats[:n].cpu().numpy(), ref)
        assert stats.cpu().numpy().tolist() == oracle.lookup_counts(dref, orc.nodes).tolist()
    c.free()


@pytest.mark.parametrize("alias", [False, True])
def test_probe_host(H, c1, c1_hot, alias):
    """helios_cache_probe_host: runs K4's host part on random host-tier rows and reports a time;
    argument and state errors are synchronous; the cache stays usable (a gather afterwards is exact)."""
    g, hot = c1_hot
    Hr, S = workloads.tier_rows(c1.cfg)
    c = H.helios_cache_build(g, hot, c1.cfg.R, Hr, S, host_table=c1.table, feature_path=c1.feature_path,
                             header_bytes=c1.header, file_stride=c1.stride, flags=H.HOST_ALIAS if alias else 0)
    ms = H.helios_cache_probe_host(c, 50_000, seed=3, reps=3)
    assert 0 < ms < 1000
    lms, depth = H.helios_cache_probe_link(c, 50_000, seed=3, reps=2)
    assert 0 < lms < 1000 and depth > 0
    assert 0 < H.helios_graph_probe_random(g, 1 << 20, reps=2) < 1000
    with pytest.raises(H.HeliosError) as e:
        H.helios_graph_probe_random(g, 0)
    assert e.value.name == "E_INVALID"
    for n, reps in ((0, 1), (10, 0)):
        with pytest.raises(H.HeliosError) as e:
            H.helios_cache_probe_host(c, n, reps=reps)
        assert e.value.name == "E_INVALID"
    dref, _ = oracle.cache_dir(hot.cpu().numpy().astype(np.uint64), 1, Hr, S, host_slot_is_id=alias)
    nodes = np.arange(c1.cfg.V, dtype=np.int64)
    gather_and_check(H, c, c1, nodes, oracle.lookup_counts(dref, nodes))
    c.free()
    c0 = H.helios_cache_build(g, hot, c1.cfg.R, c1.cfg.V, 0, host_table=c1.table)
    with pytest.raises(H.HeliosError) as e:
        H.helios_cache_probe_host(c0, 100)
    assert e.value.name == "E_STATE"
    with pytest.raises(H.HeliosError) as e:
        H.helios_cache_probe_link(c0, 100)
    assert e.value.name == "E_STATE"
    c0.free()


def _check_batch(H, c1, blocks, feats, seeds, key):
    got = blocks.to_host()
    orc = oracle.sample(c1.graph.indptr, c1.graph.indices, seeds, c1.cfg.fanouts, key)
    assert np.array_equal(got["nodes"], orc.nodes)
    for h in range(len(c1.cfg.fanouts)):
        assert np.array_equal(got["block_indices"][h], orc.block_indices[h])
    assert np.array_equal(feats[: len(orc.nodes)].cpu().numpy(), oracle.gather(orc.nodes, c1.cfg.R, table=c1.table))


@pytest.mark.parametrize("bad", [-3, 10_005, 2**40])
def test_bad_seed_latches_range(H, c1, c1_hot, bad):
    """A seed outside [0, V) through helios_batch_prepare, helios_plan_submit (device and host seeds),
    helios_gather and helios_presample latches E_RANGE (helios.h) without any out-of-bounds access:
    the context stays healthy and the next good batch is bit-exact (memcheck: profiles/sanitizer_r02)."""
    g, hot = c1_hot
    cfg = c1.cfg
    Hr, S = workloads.tier_rows(cfg)
    c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=c1.table, feature_path=c1.feature_path,
                             header_bytes=c1.header, file_stride=c1.stride, flags=H.HOST_ALIAS)
    keys = workloads.batch_keys(0, 2)
    good = c1.batches[0]
    badseeds = good.copy()
    badseeds[7] = bad
    blocks = H.Blocks.allocate(cfg.B, cfg.fanouts, g.V, g.E)
    feats = torch.empty((blocks.nodes.numel(), cfg.R), dtype=torch.uint8, device="cuda")
    H.helios_batch_prepare(g, c, torch.as_tensor(badseeds).cuda(), cfg.fanouts, keys[0], blocks, feats)
    with pytest.raises(H.HeliosError) as e:
        H.helios_sync(c)
    assert e.value.name == "E_RANGE"
    H.helios_batch_prepare(g, c, torch.as_tensor(good).cuda(), cfg.fanouts, keys[1], blocks, feats)
    H.helios_sync(c)
    _check_batch(H, c1, blocks, feats, good, keys[1])
    # the plan (CUDA graphs), device seeds and host seeds
    plan = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=2)
    dev_bad = torch.as_tensor(badseeds).cuda()
    for k, sd in enumerate((dev_bad, badseeds)):
        H.helios_plan_submit(plan, k, sd, keys[0])
        H.helios_plan_wait(plan, k)
        with pytest.raises(H.HeliosError) as e:
            H.helios_sync(c)
        assert e.value.name == "E_RANGE"
    H.helios_plan_submit(plan, 0, good, keys[1])
    H.helios_plan_wait(plan, 0)
    H.helios_sync(c)
    blk, fts, _ = plan.outputs[0]
    _check_batch(H, c1, blk, fts, good, keys[1])
    plan.free()
    # helios_gather of a bad id
    out = torch.empty((4, cfg.R), dtype=torch.uint8, device="cuda")
    H.helios_gather(c, torch.tensor([1, bad, 2, 3], device="cuda"), torch.tensor([4], device="cuda"), out)
    with pytest.raises(H.HeliosError) as e:
        H.helios_sync(c)
    assert e.value.name == "E_RANGE"
    c.free()
    # presample of a bad seed: latched, no out-of-bounds hotness update
    hot2 = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
    H.helios_presample(g, torch.as_tensor(badseeds).cuda(), cfg.B, cfg.fanouts, [keys[0]], hot2)
    with pytest.raises(H.HeliosError) as e:
        H.helios_graph_sync(g)
    assert e.value.name == "E_RANGE"
    assert int(hot2.sum()) > 0


def test_seed_dtype_conversion(H, c1, c1_hot):
    """int32 / non-contiguous seeds are converted by the binding (never read as int64 past the end)."""
    g, hot = c1_hot
    cfg = c1.cfg
    c = H.helios_cache_build(g, hot, cfg.R, cfg.V, 0, host_table=c1.table)
    keys = workloads.batch_keys(0, 1)
    good = c1.batches[0]
    plan = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=1)
    s32 = torch.as_tensor(good.astype(np.int32)).cuda()
    H.helios_plan_submit(plan, 0, s32, keys[0])
    H.helios_plan_wait(plan, 0)
    H.helios_sync(c)
    blk, fts, _ = plan.outputs[0]
    _check_batch(H, c1, blk, fts, good, keys[0])
    plan.free()
    blocks = H.Blocks.allocate(cfg.B, cfg.fanouts, g.V, g.E)
    feats = torch.empty((blocks.nodes.numel(), cfg.R), dtype=torch.uint8, device="cuda")
    strided = torch.as_tensor(np.repeat(good, 2)).cuda()[::2]
    H.helios_batch_prepare(g, c, strided.to(torch.int32), cfg.fanouts, keys[0], blocks, feats)
    H.helios_sync(c)
    _check_batch(H, c1, blocks, feats, good, keys[0])
    c.free()
