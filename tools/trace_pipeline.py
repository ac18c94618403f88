"""Pipeline timeline from the device-side tracer (HELIOS_PLAN_TRACE): for C2 / C3 at depth 8, the
mean duration of every kernel position, the gap between a kernel and its predecessor in the batch's
chain (dependency + launch latency), the batch latency, how many batches each kernel position
overlaps with on average, and the throughput with tracing on and off.  One JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
os.environ.setdefault("HELIOS_LIB", "trace")
from paper_2310_00837_b200 import helios as H  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 8
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
seeds = {b: torch.as_tensor(inp.batches[b]).cuda() for b in full}
L = len(cfg.fanouts)
names = [f"{k}_h{h}" for h in range(L) for k in ("count_scan", "fill", "assign")] + ["relabel", "table_clear",
                                                                                     "lookup", "gather"]
out = {"config": cfg.name, "depth": depth}
n = 1600
for flags, tag in ((0, "off"), (H.PLAN_TRACE, "on")):
    p = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=depth, flags=flags)
    sub = lambda i: H.helios_plan_submit(p, i % depth, seeds[full[i % len(full)]], keys[full[i % len(full)]])
    for i in range(64):
        sub(i)
    torch.cuda.synchronize()
    a, bev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        sub(i)
    for k in range(depth):
        H.helios_plan_wait(p, k)
    bev.record()
    bev.synchronize()
    out[f"batches_s_trace_{tag}"] = round(n / (a.elapsed_time(bev) / 1e3))
    if flags:
        rows = []
        for k in range(depth):
            for back in range(min(n // depth, 200)):
                rows.append(H.helios_plan_trace(p, k, back).astype(np.int64))
        T = np.stack(rows)                     # [batches, K, 2]
        dur = (T[:, :, 1] - T[:, :, 0]) / 1e3  # us
        gap = (T[:, 1:, 0] - T[:, :-1, 1]) / 1e3
        lat = (T[:, -1, 1] - T[:, 0, 0]) / 1e3
        # overlap: how many other batches' intervals of any kernel intersect this kernel's interval
        t0, t1 = T[:, :, 0].min(), T[:, :, 1].max()
        span_us = (t1 - t0) / 1e3
        busy = {}
        for kk, nm in enumerate(names):
            busy[nm] = round(float(dur[:, kk].sum()) / span_us, 3)   # mean instances of this kernel running
        out["kernels"] = {nm: {"mean_us": round(float(dur[:, kk].mean()), 2),
                               "gap_before_us": round(float(gap[:, kk - 1].mean()), 2) if kk else None,
                               "mean_concurrent": busy[nm]} for kk, nm in enumerate(names)}
        out["batch_latency_us"] = round(float(lat.mean()), 1)
        out["sum_kernel_us"] = round(float(dur.sum(axis=1).mean()), 1)
        out["sum_gaps_us"] = round(float(gap.sum(axis=1).mean()), 1)
        out["batches_traced"] = len(rows)
    p.free()
print(json.dumps(out))
