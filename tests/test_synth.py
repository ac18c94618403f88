"""Input-generator checks (synth/): SplitMix64 golden values, permutation bijection, CSR validity
(indptr[0]=0, monotone, indptr[V]=E, indices < V), no self-loops or multi-edges,
determinism, 1% training set, epoch batches partition the training set."""
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_mix64_golden():
    for line in open(os.path.join(GOLD, "splitmix64.txt")):
        if line.startswith("#") or not line.strip():
            continue
        x, y = (int(t, 16) for t in line.split())
        assert synth.mix64(x) == y


@pytest.mark.parametrize("scale", [3, 10, 14])
def test_perm_bijection(scale):
    L = synth.lib()
    ys = [L.synth_perm_fwd(scale, 77, x) for x in range(1 << scale)]
    assert sorted(ys) == list(range(1 << scale))
    assert all(L.synth_perm_inv(scale, 77, y) == x for x, y in enumerate(ys))


def test_graph_valid_and_deterministic():
    g = synth.graph(5000, 80000, seed=9)
    ip, ix = g.indptr, g.indices
    assert ip[0] == 0 and np.all(np.diff(ip) >= 0) and ip[-1] == len(ix)
    assert ix.min() >= 0 and ix.max() < g.V
    for v in range(g.V):
        row = ix[ip[v]:ip[v + 1]]
        assert np.all(np.diff(row) > 0) and not np.any(row == v)
    g2 = synth.graph(5000, 80000, seed=9)
    assert np.array_equal(g.indptr, g2.indptr) and np.array_equal(g.indices, g2.indices)
    st = g.degree_stats()
    assert st["max_in_deg"] > 20 * st["avg_deg"]   # power-law skew


def test_train_and_batches():
    tr = synth.train_set(100000)
    assert 800 < len(tr) < 1200 and np.all(np.diff(tr) > 0)
    bs = synth.epoch_batches(tr, 128, epoch=3)
    allv = np.concatenate(bs)
    assert np.array_equal(np.sort(allv), tr)
    assert all(len(b) == 128 for b in bs[:-1])
    assert not np.array_equal(np.concatenate(synth.epoch_batches(tr, 128, epoch=4)), allv)
