"""Pins for oracle.sample (ORACLE_SAMPLE; "random neighbor sampling").

* f = -1 reduces to breadth-first discovery order from the seeds (scipy.sparse.csgraph BFS from a
  super-source whose adjacency is the seed list), truncated at depth L; blocks = CSR rows relabelled.
* Closed forms: star, directed path, isolated seed, hub.
* On generated power-law graphs: exact fanout bound, every sampled edge exists in the CSR,
  no repeated position per row, dedup/relabel invariants (prefix, distinct, range,
  first-occurrence order).
* Error cases: duplicate seed (E_INVALID), seed out of range (E_RANGE).
"""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import breadth_first_order, shortest_path

import oracle
import synth


def csr_from_adj(adj):
    indptr = np.zeros(len(adj) + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(a) for a in adj])
    indices = np.array([u for a in adj for u in a], dtype=np.int32)
    return indptr, indices


@pytest.fixture(scope="module")
def g1():
    return synth.graph(3000, 40000, seed=11)


def check_invariants(indptr, indices, seeds, fanouts, b):
    L = len(fanouts)
    N = b.nodes
    lc = b.level_counts
    assert lc[0] == len(seeds) and np.array_equal(N[: len(seeds)], seeds)
    assert len(np.unique(N)) == len(N)                      # distinct
    for h in range(L):
        nh, nh1 = int(lc[h]), int(lc[h + 1])
        bp, bi = b.block_indptr[h], b.block_indices[h]
        assert len(bp) == nh + 1 and bp[0] == 0 and bp[-1] == len(bi) == b.edge_counts[h]
        deg = indptr[N[:nh] + 1] - indptr[N[:nh]]
        k = deg if fanouts[h] < 0 else np.minimum(deg, fanouts[h])
        assert np.array_equal(np.diff(bp), k)              # exact fanout bound
        assert bi.min(initial=0) >= 0 and bi.max(initial=-1) < nh1  # local ids in range
        # first-occurrence order of new ids: scanning block indices in (row, slot) order, each id
        # >= n_h first appears as exactly the next unused id.
        nxt = nh
        for x in bi:
            if x >= nxt:
                assert x == nxt
                nxt += 1
        assert nxt == nh1
        # edge existence + distinct positions per row (the generator emits no multi-edges)
        for i in range(nh):
            v = N[i]
            row = set(indices[indptr[v]:indptr[v + 1]].tolist())
            got = N[bi[bp[i]:bp[i + 1]]]
            assert len(set(got.tolist())) == len(got)
            assert set(got.tolist()) <= row


@pytest.mark.parametrize("fanouts", [[10, 5], [15, 10, 5], [25, 10], [3], [40]])
def test_invariants_generated(g1, fanouts):
    tr = synth.train_set(g1.V, pct=5)
    seeds = synth.epoch_batches(tr, 64, epoch=0)[0]
    b = oracle.sample(g1.indptr, g1.indices, seeds, fanouts, key=synth.batch_key(1, 0, 0))
    check_invariants(g1.indptr, g1.indices, seeds, fanouts, b)


def test_determinism_and_key_dependence(g1):
    seeds = np.arange(0, 3000, 37)
    a = oracle.sample(g1.indptr, g1.indices, seeds, [10, 5], key=99)
    b = oracle.sample(g1.indptr, g1.indices, seeds, [10, 5], key=99)
    c = oracle.sample(g1.indptr, g1.indices, seeds, [10, 5], key=100)
    assert np.array_equal(a.nodes, b.nodes)
    assert not np.array_equal(a.nodes, c.nodes)


@pytest.mark.parametrize("L", [1, 2, 3])
def test_full_fanout_is_bfs_order(g1, L):
    V = g1.V
    seeds = np.array([5, 1000, 17, 2999, 42], dtype=np.int64)
    b = oracle.sample(g1.indptr, g1.indices, seeds, [-1] * L, key=0)
    # super-source S = V with adjacency = seeds (in order)
    indptr = np.concatenate([g1.indptr, [g1.indptr[-1] + len(seeds)]])
    indices = np.concatenate([g1.indices, seeds.astype(np.int32)])
    A = sp.csr_matrix((np.ones(len(indices)), indices, indptr), shape=(V + 1, V + 1))
    order = breadth_first_order(A, V, directed=True, return_predecessors=False)
    depth = shortest_path(A, unweighted=True, directed=True, indices=V)
    keep = [u for u in order[1:] if depth[u] <= L + 1]
    assert np.array_equal(b.nodes, np.array(keep))
    # block h, row i = CSR row of N_h[i] mapped to local ids, in CSR order
    pos = {int(u): i for i, u in enumerate(b.nodes)}
    for h in range(L):
        for i in range(int(b.level_counts[h])):
            v = b.nodes[i]
            row = g1.indices[g1.indptr[v]:g1.indptr[v + 1]]
            got = b.block_indices[h][b.block_indptr[h][i]:b.block_indptr[h][i + 1]]
            assert [pos[int(u)] for u in row] == got.tolist()


def test_star_closed_forms():
    m = 50
    adj = [list(range(1, m + 1))] + [[] for _ in range(m)]
    indptr, indices = csr_from_adj(adj)
    b = oracle.sample(indptr, indices, [0], [m], key=3)
    assert b.nodes.tolist() == list(range(m + 1))        # f >= m: centre then leaves in CSR order
    b = oracle.sample(indptr, indices, [0], [7], key=3)
    assert len(b.nodes) == 8 and len(set(b.nodes[1:].tolist())) == 7 and set(b.nodes[1:].tolist()) <= set(range(1, m + 1))
    assert b.block_indices[0].tolist() == list(range(1, 8))


def test_path_and_isolated():
    n = 20
    adj = [[v + 1] for v in range(n - 1)] + [[]]
    indptr, indices = csr_from_adj(adj)
    b = oracle.sample(indptr, indices, [3], [2, 2, 2, 2], key=1)
    assert b.nodes.tolist() == [3, 4, 5, 6, 7]
    b = oracle.sample(indptr, indices, [n - 1], [5, 5], key=1)    # isolated seed: empty rows
    assert b.nodes.tolist() == [n - 1] and b.block_indptr[0].tolist() == [0, 0]


def test_hub_row():
    d = 10**6
    adj = [list(range(1, d + 1))] + [[] for _ in range(d)]
    indptr, indices = csr_from_adj(adj)
    b = oracle.sample(indptr, indices, [0], [15], key=77)
    assert len(b.nodes) == 16 and len(set(b.nodes.tolist())) == 16


def test_errors(g1):
    with pytest.raises(oracle.OracleError) as e:
        oracle.sample(g1.indptr, g1.indices, [1, 2, 1], [5], key=0)
    assert e.value.code == oracle.E_INVALID
    with pytest.raises(oracle.OracleError) as e:
        oracle.sample(g1.indptr, g1.indices, [1, g1.V], [5], key=0)
    assert e.value.code == oracle.E_RANGE


def test_star_uniformity_through_sampler():
    # each of 100 leaves is picked with frequency f/d = .25, over 8000 batch keys
    m, f, trials = 100, 25, 8000
    adj = [list(range(1, m + 1))] + [[] for _ in range(m)]
    indptr, indices = csr_from_adj(adj)
    hits = np.zeros(m + 1)
    for t in range(trials):
        b = oracle.sample(indptr, indices, [0], [f], key=synth.batch_key(5, 0, t))
        hits[b.nodes[1:]] += 1
    freq = hits[1:] / trials
    assert np.all(np.abs(freq - 0.25) < 0.025)
