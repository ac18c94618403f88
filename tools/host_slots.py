"""Host-tier access-locality study (C3): dump the host-tier slots every batch reads, plus page stats.

The host tier is packed in hot-rank order (reading 9), so slot = hot_rank - H.  This needs only the
graph and the presample pass (no feature table, no pinned tier): the hot-rank permutation is
recomputed here with torch's stable sort, which is the same order helios_cache_build produces
(hot desc, id asc).  Output: <out>.npz with `slots` (int64, concatenated) and `offs` (per batch),
consumed by tools/hostorder.cu; page statistics are printed as one JSON line.
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2310_00837_b200 import helios as H  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "/tmp/c3_slots"
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 96
    cfg = workloads.CONFIGS["C3"]
    t0 = time.time()
    inp = workloads.make_inputs(cfg, table=False)
    g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices)
    hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
    pkeys = workloads.presample_keys(len(inp.batches))
    for b in range(len(inp.batches)):
        H.helios_presample(g, torch.as_tensor(inp.batches[b]).cuda(), cfg.B, cfg.fanouts, [pkeys[b]], hot)
    H.helios_graph_sync(g)
    Hr, S = workloads.tier_rows(cfg)
    order = torch.sort(-hot, stable=True).indices
    rank = torch.empty_like(order)
    rank[order] = torch.arange(cfg.V, device="cuda")
    keys = workloads.batch_keys(0, len(inp.batches))
    full = [b for b in range(len(inp.batches)) if len(inp.batches[b]) == cfg.B][:nb]
    blk = H.Blocks.allocate(cfg.B, cfg.fanouts, cfg.V, inp.graph.E)
    slots, offs = [], [0]
    for b in full:
        H.helios_sample(g, torch.as_tensor(inp.batches[b]).cuda(), cfg.fanouts, keys[b], blk)
        torch.cuda.synchronize()
        n = int(blk.level_counts[len(cfg.fanouts)].item())
        r = rank[blk.nodes[:n]]
        s = (r[(r >= Hr) & (r < Hr + S)] - Hr).cpu().numpy()
        slots.append(s)
        offs.append(offs[-1] + len(s))
    allv = np.concatenate(slots)
    np.savez(out, slots=allv, offs=np.asarray(offs, dtype=np.int64), R=cfg.R, S=S)
    allv.astype(np.int64).tofile(out + ".slots.bin")
    np.asarray(offs, dtype=np.int64).tofile(out + ".offs.bin")
    R = cfg.R
    st = {"batches": len(full), "host_rows_per_batch": float(np.mean([len(s) for s in slots]))}
    for name, sh in (("4KB", 12), ("64KB", 16), ("2MB", 21), ("1GB", 30)):
        per = [len(np.unique((s * R) >> sh)) for s in slots]
        st[f"distinct_{name}_pages_per_batch"] = float(np.mean(per))
        w6 = [len(np.unique((np.concatenate(slots[i:i + 6]) * R) >> sh)) for i in range(0, len(slots) - 5, 6)]
        st[f"distinct_{name}_pages_per_6_batches"] = float(np.mean(w6))
    q = np.quantile(allv, [0.1, 0.25, 0.5, 0.75, 0.9]) * R / 2**30
    st["slot_quantiles_GB"] = [round(float(x), 2) for x in q]
    st["setup_s"] = round(time.time() - t0, 1)
    print(json.dumps(st))


if __name__ == "__main__":
    main()
