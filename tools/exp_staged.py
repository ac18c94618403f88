"""Experiment: the staged host tier's dynamic split, K3+K4 alone on real sampled lists (C3 shape,
scale from argv), for several caches: zero-copy, and staged with stage_frac caps / stager counts.
Prints one JSON line per variant: ms per gather, host rows per batch, rows the stagers copied."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from paper_2310_00837_b200 import helios as H  # noqa: E402

s = float(sys.argv[1]) if len(sys.argv) > 1 else 0.25
cfg = workloads.scaled(workloads.CONFIGS["C3"], s)
inp = workloads.make_inputs(cfg, table=True)
g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices)
hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
pk = workloads.presample_keys(len(inp.batches))
for b in range(len(inp.batches)):
    H.helios_presample(g, torch.as_tensor(inp.batches[b]).cuda(), cfg.B, cfg.fanouts, [pk[b]], hot)
H.helios_graph_sync(g)
Hr, S = workloads.tier_rows(cfg)
keys = workloads.batch_keys(0, len(inp.batches))
full = [b for b in range(len(inp.batches)) if len(inp.batches[b]) == cfg.B]
L = len(cfg.fanouts)
blks = []
for j in range(16):
    bb = full[j % len(full)]
    blk = H.Blocks.allocate(cfg.B, cfg.fanouts, cfg.V, inp.graph.E)
    H.helios_sample(g, torch.as_tensor(inp.batches[bb]).cuda(), cfg.fanouts, keys[bb], blk)
    blks.append((bb, blk))
torch.cuda.synchronize()
variants = [("zero-copy", 0, 0.0, 0)] + [(f"staged w{w} f{f}", H.HOST_STAGED, f, w)
                                        for (w, f) in ((8, 0.02), (8, 0.5), (8, 1.0), (2, 1.0), (16, 1.0))]
only = os.environ.get("EXP_VARIANTS")   # e.g. "0,3": run only these variants
if only:
    variants = [variants[int(k)] for k in only.split(",")]
for name, flags, frac, workers in variants:
    c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=inp.table, flags=flags, stage_frac=frac,
                             stage_workers=workers)
    feats = torch.empty((blks[0][1].nodes.numel(), cfg.R), dtype=torch.uint8, device="cuda")
    stats = H.new_stats()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times, host = [], 0
    for rep in range(3):
        for bb, blk in blks:
            torch.cuda.synchronize()
            ev0.record()
            H.helios_gather(c, blk.nodes, blk.level_counts[L:L + 1], feats, stats)
            ev1.record()
            ev1.synchronize()
            H.helios_sync(c)
            times.append(ev0.elapsed_time(ev1))
            host += int(stats[2].item())
    bb, blk = blks[-1]
    orc = oracle.sample(inp.graph.indptr, inp.graph.indices, inp.batches[bb], cfg.fanouts, keys[bb])
    ok = bool(np.array_equal(feats[: len(orc.nodes)].cpu().numpy(), oracle.gather(orc.nodes, cfg.R, table=inp.table)))
    inf = c.info()
    print(json.dumps({"variant": name, "scale": s, "ms_median": round(float(np.median(times)), 4),
                      "ms_min": round(float(np.min(times)), 4), "ms_max": round(float(np.max(times)), 4),
                      "host_rows_per_batch": host / len(times), "staged_rows_per_batch": inf.staged_rows / len(times),
                      "parity": ok}), flush=True)
    c.free()
