"""Experiment: sampling-only plan throughput (depth 8, CUDA graphs) on the C2 / C3 graph for the
fanout prefixes [15], [15,10], [15,10,5] -- the marginal GPU cost of each hop.  One JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2310_00837_b200 import helios as H  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
inp = workloads.make_inputs(cfg, table=False)
g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices)
keys = workloads.batch_keys(0, len(inp.batches))
full = [b for b in range(len(inp.batches)) if len(inp.batches[b]) == cfg.B]
seeds = {b: torch.as_tensor(inp.batches[b]).cuda() for b in full}
depth, n = int(os.environ.get("DEPTH", "8")), 3000
out = {"config": cfg.name}
for fan in ([15], [15, 10], [15, 10, 5]):
    p = H.helios_plan_create(g, None, cfg.B, fan, depth=depth)
    sub = lambda i: H.helios_plan_submit(p, i % depth, seeds[full[i % len(full)]], keys[full[i % len(full)]])
    for i in range(40):
        sub(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        sub(i)
    for k in range(depth):
        H.helios_plan_wait(p, k)
    b.record()
    b.synchronize()
    lc = p.outputs[0][0].level_counts.cpu().tolist()
    out[str(fan)] = {"batches_s": round(n / (a.elapsed_time(b) / 1e3)), "us_per_batch": round(a.elapsed_time(b) * 1e3 / n, 2),
                     "level_counts_last": lc}
    p.free()
print(json.dumps(out))
