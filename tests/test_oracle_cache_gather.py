"""Pins for oracle.presample / cache_dir / lookup_counts / gather.

* presample == brute-force recount: a Python set union over each presample batch's N_L.
* cache_dir: the ordering equals numpy's stable lexsort by (hot desc, id asc); tier-order
  invariant min hot(HBM) >= max hot(HOST) >= max hot(FILE); exact tier caps; all-equal hotness
  gives tiers by ascending id; owner = rank mod G, slot = rank div G.
* lookup_counts == numpy tally of decoded directory words.
* gather: bytes equal the synth_feature closed form recomputed in pure Python integer arithmetic,
  equal the file bytes, and tiers-on (FILE rows via pread) == tiers-off.
"""
import os
import struct

import numpy as np
import pytest

import oracle
import synth


@pytest.fixture(scope="module")
def g():
    return synth.graph(4000, 60000, seed=3)


def test_presample_bruteforce(g):
    tr = synth.train_set(g.V, pct=5)
    batches = synth.epoch_batches(tr, 50, epoch=0)
    keys = [synth.presample_key(7, b) for b in range(len(batches))]
    hot = oracle.presample(g.indptr, g.indices, batches, keys, [10, 5])
    ref = np.zeros(g.V, dtype=np.uint64)
    for s, k in zip(batches, keys):
        for v in set(oracle.sample(g.indptr, g.indices, s, [10, 5], k).nodes.tolist()):
            ref[v] += 1
    assert np.array_equal(hot, ref)


def test_cache_dir_order_and_tiers(g):
    rng = np.random.default_rng(0)
    hot = rng.integers(0, 30, g.V).astype(np.uint64)
    for G, H, S, alias in [(1, 400, 1600, False), (4, 100, 1000, False), (3, 0, 500, True), (2, 2000, 0, False)]:
        d, order = oracle.cache_dir(hot, G, H, S, host_slot_is_id=alias)
        ids = np.arange(g.V)
        ref_order = np.lexsort((ids, -hot.astype(np.int64)))
        assert np.array_equal(order, ref_order)
        tier, owner, slot = oracle.dir_decode(d)
        rank = np.empty(g.V, dtype=np.int64)
        rank[order] = np.arange(g.V)
        assert (tier == 0).sum() == min(g.V, G * H) and (tier == 1).sum() == min(max(0, g.V - G * H), S)
        hbm = tier == 0
        assert np.array_equal(owner[hbm], rank[hbm] % G) and np.array_equal(slot[hbm], rank[hbm] // G)
        host = tier == 1
        assert np.array_equal(slot[host], ids[host] if alias else rank[host] - G * H)
        fil = tier == 2
        assert np.array_equal(slot[fil], ids[fil])
        for a, b in [(0, 1), (1, 2), (0, 2)]:
            if (tier == a).any() and (tier == b).any():
                assert hot[tier == a].min() >= hot[tier == b].max()


def test_cache_dir_all_equal(g):
    d, order = oracle.cache_dir(np.full(g.V, 5, dtype=np.uint64), 1, 100, 300)
    tier, _, slot = oracle.dir_decode(d)
    assert np.array_equal(order, np.arange(g.V))
    assert (tier[:100] == 0).all() and (tier[100:400] == 1).all() and (tier[400:] == 2).all()
    assert np.array_equal(slot[:100], np.arange(100))


def test_lookup_counts(g):
    hot = np.random.default_rng(1).integers(0, 9, g.V).astype(np.uint64)
    d, _ = oracle.cache_dir(hot, 4, 200, 1000)
    nodes = np.random.default_rng(2).choice(g.V, 1500, replace=False)
    tier, owner, _ = oracle.dir_decode(d[nodes])
    for rank in range(4):
        c = oracle.lookup_counts(d, nodes, rank)
        assert c.tolist() == [int(((tier == 0) & (owner == rank)).sum()), int(((tier == 0) & (owner != rank)).sum()),
                              int((tier == 1).sum()), int((tier == 2).sum())]


def _closed_form_row(v, dim):
    M = (1 << 64) - 1

    def mix(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)
    return b"".join(struct.pack("<f", (mix(v * dim + j) >> 40) * 2.0 ** -24) for j in range(dim))


@pytest.mark.parametrize("dim", [100, 128])
def test_gather_closed_form_file_and_tiers(tmp_path, dim):
    V, R = 3000, 4 * dim
    table = synth.features(V, dim)
    path = str(tmp_path / "feat.bin")
    stride = synth.write_feature_file(path, V, dim, header_bytes=4096)
    assert stride == (R + 511) // 512 * 512
    nodes = np.random.default_rng(dim).permutation(V)[:700]
    out_t = oracle.gather(nodes, R, table=table)
    for i in (0, 1, 350, 699):
        assert out_t[i].tobytes() == _closed_form_row(int(nodes[i]), dim)
    out_f = oracle.gather(nodes, R, path=path, header=4096, stride=stride)
    assert np.array_equal(out_t, out_f)
    hot = np.random.default_rng(3).integers(0, 5, V).astype(np.uint64)
    d, _ = oracle.cache_dir(hot, 1, 300, 1200)
    out_mixed = oracle.gather(nodes, R, table=table, path=path, header=4096, stride=stride, dir_=d)
    assert np.array_equal(out_t, out_mixed)
    # file bytes themselves: padding zero, row at header + v*stride
    with open(path, "rb") as fh:
        fh.seek(4096 + 17 * stride)
        raw = fh.read(stride)
    assert raw[:R] == _closed_form_row(17, dim) and raw[R:] == b"\0" * (stride - R)
