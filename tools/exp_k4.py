"""Experiment: K3+K4 alone on real sampled node lists (SURVEY §8(d) per-kernel roofline; VERDICT r01
next-5).  Samples 64 batches of the config once, then runs helios_gather (lookup + gather) on them
back to back on one stream, `reps` times, timed with CUDA events; prints one JSON line with the
algorithmic HBM bytes per launch and GB/s.  Variants come from the environment at cache build
(HELIOS_GATHER_CTAS_PER_SM, HELIOS_GATHER_BULK).  Run under ncu (-k regex:k_gather_lists) for the
K4-only duration and DRAM throughput."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from paper_2310_00837_b200 import helios as H  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
inp = workloads.make_inputs(cfg, table=True)
g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices)
hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
pk = workloads.presample_keys(len(inp.batches))
for b in range(len(inp.batches)):
    H.helios_presample(g, torch.as_tensor(inp.batches[b]).cuda(), cfg.B, cfg.fanouts, [pk[b]], hot)
H.helios_graph_sync(g)
Hr, S = workloads.tier_rows(cfg)
if cfg.hbm_frac + cfg.host_frac >= 1.0:
    S = max(0, cfg.V - Hr)
c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=inp.table)
keys = workloads.batch_keys(0, len(inp.batches))
full = [b for b in range(len(inp.batches)) if len(inp.batches[b]) == cfg.B]
L = len(cfg.fanouts)
blks = []
for j in range(64):
    bb = full[j % len(full)]
    blk = H.Blocks.allocate(cfg.B, cfg.fanouts, cfg.V, inp.graph.E)
    H.helios_sample(g, torch.as_tensor(inp.batches[bb]).cuda(), cfg.fanouts, keys[bb], blk)
    blks.append((bb, blk))
torch.cuda.synchronize()
feats = torch.empty((blks[0][1].nodes.numel(), cfg.R), dtype=torch.uint8, device="cuda")
stats = H.new_stats()
rows = np.zeros(4)
nL = 0
for _, blk in blks:
    H.helios_gather(c, blk.nodes, blk.level_counts[L:L + 1], feats, stats)
    H.helios_sync(c)
    rows += stats.cpu().numpy()
    nL += int(blk.level_counts[L].item())
# parity of the last gathered batch (the variant under test must be exact)
bb, blk = blks[-1]
orc = oracle.sample(inp.graph.indptr, inp.graph.indices, inp.batches[bb], cfg.fanouts, keys[bb])
ok = bool(np.array_equal(feats[: len(orc.nodes)].cpu().numpy(), oracle.gather(orc.nodes, cfg.R, table=inp.table)))
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _, blk in blks[:8]:
        H.helios_gather(c, blk.nodes, blk.level_counts[L:L + 1], feats, None, stream=st)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for r in range(reps):
        for _, blk in blks:
            H.helios_gather(c, blk.nodes, blk.level_counts[L:L + 1], feats, None, stream=st)
    e.record(st)
e.synchronize()
ms = a.elapsed_time(e) / (reps * len(blks))
n_local, n_host = rows[0] / len(blks), rows[2] / len(blks)
nLm = nL / len(blks)
hbm_bytes = cfg.R * n_local + cfg.R * nLm + 16 * nLm
print(json.dumps({"config": cfg.name, "variant": {k: os.environ.get(k) for k in ("HELIOS_GATHER_CTAS_PER_SM", "HELIOS_GATHER_BULK", "HELIOS_GATHER_VU")},
                  "n_L": round(nLm, 1), "rows_local": round(n_local, 1), "rows_host": round(n_host, 1),
                  "hbm_bytes_per_launch": round(hbm_bytes), "ms_per_gather_k3k4": round(ms, 5),
                  "hbm_gbs_k3k4": round(hbm_bytes / ms / 1e6, 1), "parity": ok}), flush=True)
