"""Experiment: where does a C2 step go?  Throughput (depth 8, CUDA graphs) of the whole batch, of a
sampling-only plan, and of gather-only launches (helios_gather on pre-sampled node lists), each on
its own, on the C2 graph with the fully HBM-cached tier.  One JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2310_00837_b200 import helios as H  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
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
depth, n = 8, 2000
out = {"config": cfg.name}


def timed(fn):
    for i in range(40):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        fn(i)
    return a, b


for name, cache in (("whole_batch", c), ("sampling_only", None)):
    p = H.helios_plan_create(g, cache, cfg.B, cfg.fanouts, depth=depth)
    a, b = timed(lambda i: H.helios_plan_submit(p, i % depth, seeds[full[i % len(full)]], keys[full[i % len(full)]]))
    for k in range(depth):
        H.helios_plan_wait(p, k)
    b.record()
    b.synchronize()
    out[name] = round(n / (a.elapsed_time(b) / 1e3))
    p.free()

# gather only: node lists of 64 sampled batches, gathered round-robin on `depth` streams
blks = []
for j in range(64):
    bb = full[j % len(full)]
    blk = H.Blocks.allocate(cfg.B, cfg.fanouts, cfg.V, inp.graph.E)
    H.helios_sample(g, seeds[bb], cfg.fanouts, keys[bb], blk)
    blks.append(blk)
torch.cuda.synchronize()
L = len(cfg.fanouts)
feats = [torch.empty((blks[0].nodes.numel(), cfg.R), dtype=torch.uint8, device="cuda") for _ in range(2)]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    a, b = timed(lambda i: H.helios_gather(c, blks[i % 64].nodes, blks[i % 64].level_counts[L:L + 1],
                                           feats[i % 2], None, stream=st))
    b.record()
b.synchronize()
out["gather_only_serial"] = round(n / (a.elapsed_time(b) / 1e3))
print(json.dumps(out))
