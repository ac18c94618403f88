"""Host-tier layout study at C3 scale (GPU box): how many distinct 64 KB / 4 KB units of the host
tier does a batch touch under (A) hot-rank order and (B) rows grouped by a "home" in-neighbour
(the in-neighbour expected to sample the row most often at the last hop), homes in hot-rank order?
Fewer distinct units = fewer host-side translation misses (profiles/iotlb_r01.jsonl)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2310_00837_b200 import helios as H  # noqa: E402


def main():
    s = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    cfg = workloads.scaled(workloads.CONFIGS["C3"], s)
    t0 = time.time()
    inp = workloads.make_inputs(cfg, table=False)
    g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices)
    V = cfg.V
    hot = torch.zeros(V, dtype=torch.int64, device="cuda")
    pk = workloads.presample_keys(len(inp.batches))
    for b in range(len(inp.batches)):
        H.helios_presample(g, torch.as_tensor(inp.batches[b]).cuda(), cfg.B, cfg.fanouts, [pk[b]], hot)
    H.helios_graph_sync(g)
    order = torch.sort(-hot, stable=True).indices
    rank = torch.empty_like(order)
    rank[order] = torch.arange(V, device="cuda")
    Hr, S = workloads.tier_rows(cfg)
    indptr = torch.as_tensor(inp.graph.indptr).cuda()
    deg = indptr[1:] - indptr[:-1]
    # home(u) = argmax over in-edges (v -> u) of hot[v] * min(1, 5 / deg(v)), ties -> smaller v:
    # one 64-bit atomic max per edge of (quantised score << 32 | ~v), chunked over the edges
    best = torch.zeros(V, dtype=torch.int64, device="cuda")
    E = inp.graph.E
    chunk = 1 << 27
    for e0 in range(0, E, chunk):
        e1 = min(E, e0 + chunk)
        dst = torch.as_tensor(inp.graph.indices[e0:e1]).cuda().long()
        src = torch.searchsorted(indptr, torch.arange(e0, e1, device="cuda"), right=True) - 1
        sc = hot[src].double() * torch.clamp(5.0 / torch.clamp(deg[src], min=1).double(), max=1.0)
        q = torch.clamp((sc * 1024).long(), max=(1 << 30) - 1)
        key = (q << 32) | ((~src) & 0xFFFFFFFF)
        best.scatter_reduce_(0, dst, key, reduce="amax")
    home = torch.where(best > 0, (~(best & 0xFFFFFFFF)) & 0xFFFFFFFF, torch.full_like(best, -1))
    host = (rank >= Hr) & (rank < Hr + S)
    hv = torch.nonzero(host).squeeze(1)
    hk = torch.where(home[hv] >= 0, rank[home[hv].clamp(min=0)], V + rank[hv])
    kb = hk * (2 * V) + rank[hv]
    ob = hv[torch.sort(kb).indices]
    slotB = torch.full((V,), -1, dtype=torch.int64, device="cuda")
    slotB[ob] = torch.arange(len(ob), device="cuda")
    slotA = torch.where(host, rank - Hr, torch.full_like(rank, -1))
    print("setup", round(time.time() - t0, 1), flush=True)
    keys = workloads.batch_keys(0, len(inp.batches))
    blk = H.Blocks.allocate(cfg.B, cfg.fanouts, V, E)
    R = cfg.R
    res = {"A_hot_rank": [[], []], "B_home_grouped": [[], []]}
    win = {"A_hot_rank": [], "B_home_grouped": []}
    for b in range(nb):
        H.helios_sample(g, torch.as_tensor(inp.batches[b]).cuda(), cfg.fanouts, keys[b], blk)
        torch.cuda.synchronize()
        n = int(blk.level_counts[len(cfg.fanouts)].item())
        nodes = blk.nodes[:n]
        m = host[nodes]
        for name, sl in (("A_hot_rank", slotA), ("B_home_grouped", slotB)):
            sv = sl[nodes[m]]
            res[name][0].append(len(torch.unique((sv * R) >> 16)))
            res[name][1].append(len(torch.unique((sv * R) >> 12)))
            win[name].append(sv)
    out = {"scale": s, "batches": nb, "host_rows_per_batch": float(np.mean([len(x) for x in win["A_hot_rank"]]))}
    for name in res:
        w = [len(torch.unique((torch.cat(win[name][i:i + 8]) * R) >> 16)) for i in range(0, nb - 7, 8)]
        out[name] = {"distinct_64KB_per_batch": float(np.mean(res[name][0])), "distinct_4KB_per_batch": float(np.mean(res[name][1])),
                     "distinct_64KB_per_8_batches": float(np.mean(w))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
