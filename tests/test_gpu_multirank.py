"""The N>1 path on one GPU: 2 ranks as 2 processes on cuda:0 (CUDA IPC works across processes on
the same device), gloo for the setup collectives.  Each rank builds its HBM shard (G=2), the packed
host tier is one /dev/shm mapping filled by rank 0, blobs are all-gathered and peer shards attached;
every rank's batches (b = rank mod 2) must equal the oracle bit for bit, and its per-tier counts
(local / peer / host / file) must equal the oracle's lookup_counts for that rank.  The C5-rep ablation
(HELIOS_CACHE_HBM_REPLICATED: every rank holds the same hottest rows) runs the same checks against the
single-GPU directory and must read no peer rows."""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tag, q, replicated, hbm_only=False):
    import faulthandler
    faulthandler.dump_traceback_later(100, exit=True)
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import oracle
        import synth
        import workloads
        from paper_2310_00837_b200 import dist as hd
        from paper_2310_00837_b200 import helios as H
        cfg = workloads.Config("mr", 60_000, 900_000, 64, 256, [10, 5], 0.1, 0.9, train_pct=5)
        inp = workloads.make_inputs(cfg, table=True)
        g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices)
        pk = workloads.presample_keys(len(inp.batches))
        hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
        for b in hd.rank_batches(len(inp.batches), rank, world):
            H.helios_presample(g, torch.as_tensor(inp.batches[b]).cuda(), cfg.B, cfg.fanouts, [pk[b]], hot)
        H.helios_graph_sync(g)
        hot_cpu = hot.cpu()
        hd.allreduce_hotness(hot_cpu)
        hot.copy_(hot_cpu)
        Hr = int(0.1 * cfg.V)
        G = 1 if replicated else world   # the directory's world size
        S = cfg.V - G * Hr
        rf = H.HBM_REPLICATED if replicated else 0
        name = f"helios_mr_{tag}"
        if hbm_only:   # every row in the (sharded) HBM tier: the fused lookup + gather path with peer rows
            Hr, S = -(-cfg.V // world), 0
            c = H.helios_cache_build(g, hot, cfg.R, Hr, 0, host_table=inp.table, world_size=world, rank=rank)
        elif rank == 0:   # creator first, then the others map it (after the barrier)
            tier, m = hd.shared_array(name, (S * cfg.R,), np.uint8, create=True)
            c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=inp.table, world_size=world, rank=rank,
                                     host_tier=tier, flags=H.HOST_FILL | rf)
        dist.barrier()
        if rank != 0 and not hbm_only:
            tier, m = hd.shared_array(name, (S * cfg.R,), np.uint8, create=False)
            c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=inp.table, world_size=world, rank=rank,
                                     host_tier=tier, flags=rf)
        info = c.info()
        assert info.world_size == world and info.rank == rank
        print(f"[rank {rank}] cache built", file=sys.stderr, flush=True)
        hd.attach_peers(H, c)
        print(f"[rank {rank}] peers attached", file=sys.stderr, flush=True)
        dref, _ = oracle.cache_dir(hot_cpu.numpy().astype(np.uint64), G, Hr, S)
        p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=2)
        keys = workloads.batch_keys(0, len(inp.batches))
        mine = hd.rank_batches(len(inp.batches), rank, world)
        ok, peer_rows = True, 0
        for j, b in enumerate(mine):
            k = j % 2
            sd = torch.as_tensor(inp.batches[b]).cuda()   # alive until the batch completes
            H.helios_plan_submit(p, k, sd, keys[b])
            H.helios_plan_wait(p, k)
            H.helios_sync(c)
            blocks, feats, stats = p.outputs[k]
            got = blocks.to_host()
            orc = oracle.sample(inp.graph.indptr, inp.graph.indices, inp.batches[b], cfg.fanouts, keys[b])
            ok &= np.array_equal(got["nodes"], orc.nodes)
            ok &= np.array_equal(feats[: len(orc.nodes)].cpu().numpy(), oracle.gather(orc.nodes, cfg.R, table=inp.table))
            st = stats.cpu().tolist()
            ok &= st == oracle.lookup_counts(dref, orc.nodes, 0 if replicated else rank).tolist()
            peer_rows += st[1]
        print(f"[rank {rank}] batches done", file=sys.stderr, flush=True)
        dist.barrier()
        p.free()
        c.free()
        dist.barrier()
        if rank == 0 and not hbm_only:
            hd.unlink_shared(name)
        q.put((rank, bool(ok), peer_rows, len(mine)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("replicated,hbm_only", [(False, False), (True, False), (False, True)],
                         ids=["sharded", "replicated", "hbm_only_sharded"])
def test_two_ranks_one_gpu(replicated, hbm_only):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tag = f"{os.getpid()}_{port}"
    ps = [ctx.Process(target=_worker, args=(r, 2, port, tag, q, replicated, hbm_only)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=150) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, peer_rows, nb in res:
        assert ok, f"rank {rank} differs from the oracle"
        assert nb > 0
        if replicated:
            assert peer_rows == 0, f"rank {rank} read peer rows from a replicated HBM tier"
        else:
            assert peer_rows > 0, f"rank {rank} read no peer rows"
