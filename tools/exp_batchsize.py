"""Experiment: plan throughput vs batch size on the C2 graph (is the sampling chain launch-bound?)."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, synth
from paper_2310_00837_b200 import helios as H

cfg = workloads.CONFIGS["C2"]
inp = workloads.make_inputs(cfg, table=True)
g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices)
hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
c = H.helios_cache_build(g, hot, cfg.R, cfg.V, 0, host_table=inp.table)
tr = inp.train
out = {}
for B in [int(x) for x in sys.argv[1].split(",")]:
    for depth in (1, 6):
        p = H.helios_plan_create(g, c, B, cfg.fanouts, depth=depth)
        seeds = [torch.as_tensor(tr[i * B:(i + 1) * B]).cuda() for i in range(16)]
        for i in range(50):
            H.helios_plan_submit(p, i % depth, seeds[i % 16], i)
        torch.cuda.synchronize()
        n = 3000
        t0 = time.perf_counter()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(n):
            H.helios_plan_submit(p, i % depth, seeds[i % 16], i)
        for k in range(depth):
            H.helios_plan_wait(p, k)
        b.record(); b.synchronize()
        wall = time.perf_counter() - t0
        out[f"B{B}_d{depth}"] = {"batches_s": round(n / (a.elapsed_time(b) / 1e3)), "wall_batches_s": round(n / wall)}
        p.free()
print(json.dumps(out))
