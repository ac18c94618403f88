"""Host logic of the N>1 path on CPU: gloo, world_size 2.

* batches are partitioned across ranks (every batch exactly once, b = rank mod N);
* the hotness all-reduce of per-rank presample passes equals the oracle's single-pass hotness;
* the cache-export blob all-gather returns every rank's blob in rank order;
* /dev/shm shared buffers written by rank 0 are seen by rank 1.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tag, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        import workloads
        from paper_2310_00837_b200 import dist as hd
        g = synth.graph(3000, 40000, seed=2)
        tr = synth.train_set(g.V, pct=10)
        batches = synth.epoch_batches(tr, 32, 0)
        keys = [synth.presample_key(5, b) for b in range(len(batches))]
        mine = hd.rank_batches(len(batches), rank, world)
        hot = torch.from_numpy(oracle.presample(g.indptr, g.indices, [batches[b] for b in mine], [keys[b] for b in mine],
                                                [10, 5]).astype(np.int64))
        hd.allreduce_hotness(hot)
        blobs = hd.exchange_blobs(f"blob-of-{rank}".encode())
        name = f"helios_test_{tag}"
        if rank == 0:
            arr, m = hd.shared_array(name, (1000,), np.int64, create=True)
            arr[:] = np.arange(1000) * 3
        dist.barrier()
        if rank != 0:
            arr, m = hd.shared_array(name, (1000,), np.int64, create=False)
        ok_shm = bool(np.array_equal(arr, np.arange(1000) * 3))
        dist.barrier()
        if rank == 0:
            hd.unlink_shared(name)
        q.put((rank, mine, hot.numpy().tolist(), blobs, ok_shm))
    finally:
        dist.destroy_process_group()


def test_two_rank_setup_logic():
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tag = f"{os.getpid()}_{port}"
    ps = [ctx.Process(target=_worker, args=(r, 2, port, tag, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in ps:
        r = q.get(timeout=240)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = synth.graph(3000, 40000, seed=2)
    tr = synth.train_set(g.V, pct=10)
    batches = synth.epoch_batches(tr, 32, 0)
    keys = [synth.presample_key(5, b) for b in range(len(batches))]
    ref = oracle.presample(g.indptr, g.indices, batches, keys, [10, 5])
    assert sorted(res[0][1] + res[1][1]) == list(range(len(batches)))
    assert not set(res[0][1]) & set(res[1][1])
    for r in (0, 1):
        assert np.array_equal(np.array(res[r][2], dtype=np.uint64), ref)
        assert res[r][3] == [b"blob-of-0", b"blob-of-1"]
        assert res[r][4]
