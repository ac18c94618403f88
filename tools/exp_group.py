"""Experiment: is the C2 sampler bound by its kernel chain (per-batch launches and inter-kernel gaps)
or by its work?  Plans with larger batches (B = 1024, 2048, 4096 seeds, one dedup domain each) at
depths that keep the same number of seeds in flight (12 x 1024), sampling only and whole batch.
If throughput in seeds/s grows with B, grouping several batches per kernel chain pays.  One JSON
line; `eq_batches_s` = seeds/s / 1024."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2310_00837_b200 import helios as H  # noqa: E402

cfg = workloads.CONFIGS["C2"]
inp = workloads.make_inputs(cfg, table=True)
g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices)
hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
c = H.helios_cache_build(g, hot, cfg.R, cfg.V, 0, host_table=inp.table)
tr = inp.train
out = {}
n_in_flight = 12 * 1024
for B in (1024, 2048, 4096):
    chunks = [torch.as_tensor(tr[i * B:(i + 1) * B]).cuda() for i in range(len(tr) // B)]
    depth = max(1, n_in_flight // B)
    for name, cache in (("sampling_only", None), ("whole_batch", c)):
        p = H.helios_plan_create(g, cache, B, cfg.fanouts, depth=depth)
        for i in range(40):
            H.helios_plan_submit(p, i % depth, chunks[i % len(chunks)], i)
        torch.cuda.synchronize()
        n = max(300, 3000 * 1024 // B)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(n):
            H.helios_plan_submit(p, i % depth, chunks[i % len(chunks)], 1000 + i)
        for k in range(depth):
            H.helios_plan_wait(p, k)
        b.record()
        b.synchronize()
        bs = n / (a.elapsed_time(b) / 1e3)
        out[f"B{B}_d{depth}_{name}"] = {"batches_s": round(bs), "eq_batches_s": round(bs * B / 1024)}
        p.free()
print(json.dumps(out), flush=True)
