"""GPU parity of helios_sample / helios_presample (K1 sample_hop + K2 dedup_relabel) against the
CPU oracle, bit-exact: nodes (N_L), level counts, per-hop block CSR.

Sizes: the C1 config over a whole epoch; a medium power-law graph spanning many scan tiles with
ragged tails; fanout -1 (BFS), fanout > 32 (serial Floyd path), hub rows; edge cases (0/1 seeds,
isolated seeds) and the latched errors (duplicate seed, seed >= V) and E_CAPACITY.
"""
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
    assert torch.cuda.is_available()
    return helios


def run_gpu(H, g, seeds, fanouts, key):
    blocks = H.Blocks.allocate(len(seeds), fanouts, g.V, g.E)
    s = torch.as_tensor(np.asarray(seeds, dtype=np.int64)).cuda()
    H.helios_sample(g, s, fanouts, key, blocks)
    H.helios_graph_sync(g)
    return blocks.to_host()


def assert_same(gpu, orc, L):
    assert np.array_equal(gpu["level_counts"], orc.level_counts)
    assert np.array_equal(gpu["edge_counts"], orc.edge_counts)
    assert np.array_equal(gpu["nodes"], orc.nodes)
    for h in range(L):
        assert np.array_equal(gpu["block_indptr"][h], orc.block_indptr[h]), f"hop {h} indptr"
        assert np.array_equal(gpu["block_indices"][h], orc.block_indices[h]), f"hop {h} indices"


@pytest.fixture(params=["chain", "cluster", "cluster16", "tiled", "groups"])
def mode(request, monkeypatch):
    """Sampler launch mode (HELIOS_SAMPLE_MODE, read when a graph's workspace is allocated): the chain of
    2 + 3L kernels, or the whole batch in one launch of an 8- or 16-CTA cluster.  Same device code,
    so the same bits.  "tiled": the chain with the shared-memory tile dedup (HELIOS_SAMPLE_DEDUP=smem:
    per-tile shared hash, bitmap ranking, tiled relabel) for every hop with a bounded fanout.  "groups": the
    chain with the round-1 power-of-two lane groups in the fill (HELIOS_FILL_SEG=0; the default packs
    f-lane segments)."""
    chain = ("tiled", "groups")
    monkeypatch.setenv("HELIOS_SAMPLE_MODE", "chain" if request.param in chain else request.param)
    monkeypatch.delenv("HELIOS_TABLE_HOME", raising=False)
    monkeypatch.setenv("HELIOS_SAMPLE_DEDUP", "smem" if request.param == "tiled" else "global")
    monkeypatch.setenv("HELIOS_FILL_SEG", "0" if request.param == "groups" else "1")
    return request.param


@pytest.fixture(scope="module")
def c1():
    return workloads.make_inputs(workloads.CONFIGS["C1"], table=False)


@pytest.fixture(scope="module")
def medium():
    return synth.graph(300_000, 6_000_000, seed=21)


def test_c1_full_epoch(H, c1, mode):
    cfg = c1.cfg
    g = H.helios_graph_load(c1.graph.indptr, c1.graph.indices)
    keys = workloads.batch_keys(0, len(c1.batches))
    for b, (seeds, key) in enumerate(zip(c1.batches, keys)):
        gpu = run_gpu(H, g, seeds, cfg.fanouts, key)
        orc = oracle.sample(c1.graph.indptr, c1.graph.indices, seeds, cfg.fanouts, key)
        assert_same(gpu, orc, len(cfg.fanouts))


@pytest.mark.parametrize("B,fanouts", [(1024, [15, 10, 5]), (1000, [25, 10]), (333, [3, 3, 3, 3]), (77, [40]),
                                       (5, [-1, -1]), (1, [15, 10, 5])])
def test_medium_graph(H, medium, B, fanouts, mode):
    g = H.helios_graph_load(medium.indptr, medium.indices)
    rng = np.random.default_rng(B)
    seeds = rng.choice(medium.V, B, replace=False)
    for key in (1, 0xDEADBEEFCAFEF00D):
        gpu = run_gpu(H, g, seeds, fanouts, key)
        orc = oracle.sample(medium.indptr, medium.indices, seeds, fanouts, key)
        assert_same(gpu, orc, len(fanouts))


@pytest.mark.parametrize("home,medium_too", [("1024", False), ("0", True)])
def test_table_home_region(H, c1, medium, home, medium_too, monkeypatch):
    """The batch table's home region changes only where keys land, never the result: keys
    homed in the table's first 1,024 slots (C1's ~1.9 k-node batches spill past it into the worst-case table)
    or in the whole table (the round-1 hashing) give the oracle's bits.  (The default adapts the region to
    the previous batch's node count: every other test.)"""
    monkeypatch.setenv("HELIOS_TABLE_HOME", home)
    cfg = c1.cfg
    g = H.helios_graph_load(c1.graph.indptr, c1.graph.indices)
    keys = workloads.batch_keys(0, len(c1.batches))
    for b in range(0, len(c1.batches), 3):
        gpu = run_gpu(H, g, c1.batches[b], cfg.fanouts, keys[b])
        assert_same(gpu, oracle.sample(c1.graph.indptr, c1.graph.indices, c1.batches[b], cfg.fanouts, keys[b]),
                    len(cfg.fanouts))
    if not medium_too:
        return
    g = H.helios_graph_load(medium.indptr, medium.indices)
    rng = np.random.default_rng(3)
    for B, fanouts in ((1024, [15, 10, 5]), (333, [3, 3, 3, 3])):
        seeds = rng.choice(medium.V, B, replace=False)
        gpu = run_gpu(H, g, seeds, fanouts, 7)
        assert_same(gpu, oracle.sample(medium.indptr, medium.indices, seeds, fanouts, 7), len(fanouts))


def test_hub_and_isolated(H, mode, monkeypatch):
    # whole-table hashing: this test alternates 1-node and 200 k-node batches on one workspace, the adaptive
    # home region's worst case (a batch far larger than its predecessor probes long runs, DESIGN.md §5;
    # test_table_home_region covers the home regions)
    monkeypatch.setenv("HELIOS_TABLE_HOME", "0")
    d = 200_000
    adj_len = np.zeros(d + 2, dtype=np.int64)
    adj_len[0] = d
    indptr = np.concatenate([[0], np.cumsum(adj_len)])
    indices = np.arange(1, d + 1, dtype=np.int32)
    g = H.helios_graph_load(indptr, indices)
    for fan in ([15], [15, 2], [33], [-1]):
        for seeds in ([0], [0, d + 1], [d + 1], [5, 0]):
            gpu = run_gpu(H, g, seeds, fan, 12345)
            orc = oracle.sample(indptr, indices, seeds, fan, 12345)
            assert_same(gpu, orc, len(fan))


@pytest.mark.parametrize("dedup", ["global", "smem"])
def test_zero_seeds(H, c1, dedup, monkeypatch):
    monkeypatch.setenv("HELIOS_SAMPLE_DEDUP", dedup)
    g = H.helios_graph_load(c1.graph.indptr, c1.graph.indices)
    gpu = run_gpu(H, g, [], [10, 5], 1)
    assert gpu["level_counts"].tolist() == [0, 0, 0] and len(gpu["nodes"]) == 0


def test_latched_errors(H, c1):
    g = H.helios_graph_load(c1.graph.indptr, c1.graph.indices)
    with pytest.raises(H.HeliosError) as e:
        run_gpu(H, g, [1, 2, 1], [5], 1)
    assert e.value.name == "E_INVALID"
    with pytest.raises(H.HeliosError) as e:
        run_gpu(H, g, [1, c1.cfg.V + 3], [5], 1)
    assert e.value.name == "E_RANGE"
    run_gpu(H, g, [1, 2, 3], [5], 1)  # handle usable again after the latched error is read
    blocks = H.Blocks.allocate(10, [5], g.V, g.E)
    s = torch.arange(20, device="cuda", dtype=torch.int64)
    with pytest.raises(H.HeliosError) as e:
        H.helios_sample(g, s, [5], 1, blocks)
    assert e.value.name == "E_CAPACITY"


def test_graph_load_validation(H):
    with pytest.raises(H.HeliosError) as e:
        H.helios_graph_load(np.array([0, 2, 1, 3]), np.array([0, 1, 2], dtype=np.int32))
    assert e.value.name == "E_INVALID"
    with pytest.raises(H.HeliosError) as e:
        H.helios_graph_load(np.array([0, 1, 2]), np.array([0, 7], dtype=np.int32))
    assert e.value.name == "E_RANGE"


def test_presample_hotness(H, c1):
    cfg = c1.cfg
    g = H.helios_graph_load(c1.graph.indptr, c1.graph.indices)
    seeds = np.concatenate(c1.batches)
    keys = workloads.presample_keys(len(c1.batches))
    hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
    H.helios_presample(g, torch.as_tensor(seeds).cuda(), cfg.B, cfg.fanouts, keys, hot)
    H.helios_graph_sync(g)
    ref = oracle.presample(c1.graph.indptr, c1.graph.indices, c1.batches, keys, cfg.fanouts)
    assert np.array_equal(hot.cpu().numpy().astype(np.uint64), ref)


def test_persistent_sampler_parity(H, medium, monkeypatch):
    """The opt-in persistent cooperative sampler (one kernel per batch, grid barriers) is bit-exact too."""
    monkeypatch.setenv("HELIOS_SAMPLE_PERSISTENT", "1")
    g = H.helios_graph_load(medium.indptr, medium.indices)
    rng = np.random.default_rng(7)
    for B, fan in ((1024, [15, 10, 5]), (64, [40, 3]), (300, [-1])):
        seeds = rng.choice(medium.V, B, replace=False)
        gpu = run_gpu(H, g, seeds, fan, 991)
        orc = oracle.sample(medium.indptr, medium.indices, seeds, fan, 991)
        assert_same(gpu, orc, len(fan))
    g.free()


def test_host_resident_topology(H, medium, c1):
    """HELIOS_GRAPH_TOPO_HOST: the CSR in pinned host memory, sampled zero-copy over
    PCIe — same bit-exact batches and presample hotness."""
    g = H.helios_graph_load(medium.indptr, medium.indices, flags=H.GRAPH_TOPO_HOST)
    rng = np.random.default_rng(11)
    for B, fan in ((1024, [15, 10, 5]), (50, [-1, 3])):
        seeds = rng.choice(medium.V, B, replace=False)
        gpu = run_gpu(H, g, seeds, fan, 5)
        assert_same(gpu, oracle.sample(medium.indptr, medium.indices, seeds, fan, 5), len(fan))
    g.free()
    cfg = c1.cfg
    g = H.helios_graph_load(c1.graph.indptr, c1.graph.indices, flags=H.GRAPH_TOPO_HOST)
    keys = workloads.presample_keys(len(c1.batches))
    hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
    H.helios_presample(g, torch.as_tensor(np.concatenate(c1.batches)).cuda(), cfg.B, cfg.fanouts, keys, hot)
    H.helios_graph_sync(g)
    ref = oracle.presample(c1.graph.indptr, c1.graph.indices, c1.batches, keys, cfg.fanouts)
    assert np.array_equal(hot.cpu().numpy().astype(np.uint64), ref)
    with pytest.raises(H.HeliosError) as e:
        H.helios_graph_load(c1.graph.indptr, c1.graph.indices, flags=0x80)
    assert e.value.name == "E_INVALID"
