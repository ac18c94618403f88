"""bench.py — throughput of the Helios mini-batch preparation hot path on B200.

A step = one whole mini-batch through every §8(a) row: seeds -> L-hop sampling (K1/K2) -> cache
lookup + gather of N_L's feature rows from the HBM / pinned-host / file tiers (K3/K4, K5/K6).
Default workload: the papers100M-shaped config (C3; = the C5 sweep config at N=1), inputs resident
in HBM / pinned host memory before the timed region.  Under torchrun each rank takes the batches
b = rank (mod N) with its own key, the HBM tier is sharded over the ranks (peer rows over NVLink),
NCCL is used only for setup (hotness all-reduce, IPC-handle all-gather).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl helios|reference]

Prints ONE JSON line (rank 0).  See DESIGN.md §Measurement for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import mmap
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

# More hardware work queues than the default 8, so the plan's slot streams (12 in flight) and the IO /
# link streams do not alias onto shared queues (C2 +6 % at depth 12); read at CUDA context creation.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import workloads  # noqa: E402

HBM_PEAK_FALLBACK = 6650.0  # GB/s, /opt/skills/guides/B200_PROFILING.md fallback


def log(*a):
    if int(os.environ.get("RANK", "0")) == 0:
        print("[bench]", *a, file=sys.stderr, flush=True)


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def host_buffer(nbytes: int, shm_name: str | None = None, create: bool = True):
    """Page-aligned host buffer for the canonical feature table: anonymous memory with transparent
    huge pages (N=1) or a /dev/shm file shared by all ranks (N>1)."""
    if shm_name is None:
        m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        try:
            m.madvise(mmap.MADV_HUGEPAGE)
        except Exception:
            pass
        return m
    path = f"/dev/shm/{shm_name}"
    if create:
        fd = os.open(path, os.O_CREAT | os.O_RDWR | os.O_TRUNC, 0o600)
        os.ftruncate(fd, nbytes)
    else:
        fd = os.open(path, os.O_RDWR)
    m = mmap.mmap(fd, nbytes, flags=mmap.MAP_SHARED)
    os.close(fd)
    try:
        m.madvise(mmap.MADV_HUGEPAGE)
    except Exception:
        pass
    return m


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def _oneshot(self):
        try:
            return subprocess.check_output(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                            "--format=csv,noheader,nounits"], text=True, timeout=10).strip()
        except Exception:
            return ""

    def __enter__(self):
        self.first = ""
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        last = self._oneshot()
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                pass
        if last:
            self.lines.append(last)

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                for n, v in zip(names, f[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def traffic_of(name: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture."""
    d = None
    for f in ("ncu_traffic_r02.json", "ncu_traffic_r01.json"):  # latest capture of the current kernels first
        try:
            d = json.load(open(os.path.join(ROOT, "profiles", f))).get(name)
        except (OSError, ValueError):
            d = None
        if d:
            break
    if not d:
        return None
    return round(d["dram_bytes_read_per_launch"] + d["dram_bytes_write_per_launch"])


def pcie_h2d_peak(torch, nbytes: int = 1 << 30) -> float:
    """Pinned host -> device copy-engine bandwidth (GB/s, best of 5): the PCIe roofline denominator."""
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = 1e9
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        d.copy_(h, non_blocking=True)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    del h, d
    return nbytes / best / 1e6


def has_file_tier(cfg: workloads.Config) -> bool:
    return cfg.hbm_frac + cfg.host_frac < 1.0


def keeps_table(cfg: workloads.Config) -> bool:
    """The canonical host table is kept when it is small or the tiers are HBM+host only; file-tier
    configs at scale read their tier contents (and the oracle its rows) from the feature file."""
    return (not has_file_tier(cfg)) or cfg.V * cfg.R < (8 << 30)


def pick_scale(cfg: workloads.Config, world: int, workdir: str = "/tmp") -> float:
    """Capacity rule: shrink V, E by s if host RAM (canonical table, packed host tier,
    CSR) or free disk (feature file) cannot hold the config."""
    import shutil
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        return 1.0
    ram = cfg.V * cfg.R * ((1.0 if keeps_table(cfg) else 0.0) + cfg.host_frac) + cfg.E * 4 * 3 + cfg.V * 8 * 4
    s = 1.0 if ram < 0.7 * avail else 0.7 * avail / ram
    if has_file_tier(cfg):
        stride = (cfg.R + 511) // 512 * 512
        free = shutil.disk_usage(workdir).free
        s = min(s, 0.6 * free / (cfg.V * stride))
    return 1.0 if s >= 1.0 else max(0.01, math.floor(s * 100) / 100)


def file_peak(path: str, stride: int, header: int, threads: int, secs: float = 3.0) -> dict:
    """Random O_DIRECT reads of `stride` bytes with the IO workers' thread count (tools/filebench)."""
    exe = os.path.join(ROOT, "tools", "filebench")
    if not os.path.exists(exe):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-pthread", "-o", exe, exe + ".cpp"])
    out = subprocess.check_output([exe, path, str(stride), str(threads), str(secs), str(header)], text=True)
    return json.loads(out)


def sampling_accesses(batch: dict, indptr: np.ndarray, fanouts) -> dict:
    """Minimum DRAM work of one batch's sampling + lookup at 32 B sector granularity.
    Per hop and frontier row v (degree d, k = min(d, f) sampled positions): one sector for its indptr
    pair, and the sectors of indices[indptr[v] : indptr[v] + d] that hold a sampled position -- all
    S sectors of the row's span when k == d, else the expectation S * (1 - C(d - 8, k) / C(d, k)) for k
    positions drawn uniformly without replacement (8 positions per sector); one sector per node for its
    directory word.  Streaming bytes: block CSR writes (4 per edge and per indptr entry) and the node
    list (8 per node)."""
    nodes, lc = batch["nodes"], batch["level_counts"]
    sectors = stream = 0.0
    for h, f in enumerate(fanouts):
        nh = nodes[: lc[h]]
        base = indptr[nh]
        d = indptr[nh + 1] - base
        k = d if f < 0 else np.minimum(d, f)
        span = np.where(d > 0, (base + d - 1) // 8 - base // 8 + 1, 0)
        # P(no sampled position among m given positions) = C(d - m, k) / C(d, k), m = 0..8
        p_none = np.ones((9, len(nh)))
        for i in range(8):
            p_none[i + 1] = p_none[i] * np.clip((d - k - i) / np.maximum(d - i, 1), 0.0, 1.0)
        cols = np.arange(len(nh))
        m_first = np.minimum(d, 8 - base % 8)
        m_last = np.where(span > 1, base + d - 8 * ((base + d - 1) // 8), 0)
        interior = np.maximum(span - 2, 0)
        touched = ((1.0 - p_none[m_first, cols]) + np.where(span > 1, 1.0 - p_none[m_last, cols], 0.0)
                   + interior * (1.0 - p_none[8]))
        touched = np.where(k == d, span, np.where(k > 0, touched, 0.0))
        sectors += len(nh) + float(touched.sum())
        stream += 4 * int(k.sum()) + 4 * (len(nh) + 1)
    n_l = int(lc[len(fanouts)])
    sectors += n_l
    stream += 8 * n_l
    return {"sectors": sectors, "stream_bytes": stream}


def interval_union(iv) -> float:
    """Total length of the union of [a, b) intervals (ms): the time during which at least one of
    the overlapping launches was running."""
    tot, cur_a, cur_b = 0.0, None, None
    for a, b in sorted(iv):
        if cur_b is None or a > cur_b:
            if cur_b is not None:
                tot += cur_b - cur_a
            cur_a, cur_b = a, b
        else:
            cur_b = max(cur_b, b)
    if cur_b is not None:
        tot += cur_b - cur_a
    return tot


# ---------------------------------------------------------------------------------------------

def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def run_oracle_baseline(inp, keys, budget_s: float, check=None, dir_=None, threads: int = 1) -> dict:
    """The oracle as it stands (single-threaded C++ per batch), on a bounded sample of the same
    batches.  threads > 1: that many host threads, each preparing independent batches (one batch per
    thread at a time; the oracle's ctypes calls release the GIL), as SURVEY §8(d)'s P-core leg.  Rows
    come from the canonical host table, or by pread from the feature file when the config keeps no
    table (a CPU-managed cache)."""
    import oracle
    cfg = inp.cfg
    lock = threading.Lock()
    state = {"next": 0, "done": 0, "rows": 0}
    t0 = time.perf_counter()

    def worker():
        while True:
            with lock:
                b = state["next"]
                if b >= len(inp.batches) or time.perf_counter() - t0 > budget_s:
                    return
                state["next"] += 1
            ob = oracle.sample(inp.graph.indptr, inp.graph.indices, inp.batches[b], cfg.fanouts, keys[b])
            feats = oracle.gather(ob.nodes, cfg.R, table=inp.table, path=inp.feature_path, header=inp.header,
                                  stride=inp.stride, dir_=dir_)
            if check is not None:
                check(b, ob, feats)
            with lock:
                state["done"] += 1
                state["rows"] += len(ob.nodes)

    ths = [threading.Thread(target=worker) for _ in range(max(1, threads))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    return {"batches": state["done"], "seconds": dt, "value": state["done"] / dt,
            "gbs": state["rows"] * cfg.R / dt / 1e9, "threads": max(1, threads)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--scale", type=float, default=0.0, help="V,E scale factor (0 = auto from host RAM)")
    ap.add_argument("--impl", default="helios", choices=["helios", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--parity-batches", type=int, default=2)
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no baseline, no parity")
    ap.add_argument("--depth", type=int, default=0,
                    help="plan slots (groups in flight); 0 = 24 with a host tier (its gathers wait on PCIe and the "
                         "stagers, so more batches in flight pay), else 12")
    ap.add_argument("--group", type=int, default=1,
                    help="batches per plan slot: each kernel of a slot's chain launches once for its whole group "
                         "(gridDim.y); batches in flight = depth x group")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels directly instead of CUDA graphs")
    ap.add_argument("--serial-gather", type=int, default=0, help="1: gathers of successive batches run one at a time")
    ap.add_argument("--intra", action="store_true", help="intra-batch pipeline: per-hop gather passes (NEXT-1)")
    ap.add_argument("--link-stream", action="store_true",
                    help="ablation: host-tier rows of every batch on one high-priority link stream (HELIOS_PLAN_LINK_STREAM)")
    ap.add_argument("--host-alias", action="store_true", help="host tier = canonical table by id (no packed copy)")
    ap.add_argument("--io-rings", type=int, default=8, help="SQ/CQ ring pairs = host IO worker threads")
    ap.add_argument("--topo-host", action="store_true",
                    help="CSR in pinned host memory, sampled zero-copy (the paper's placement; SURVEY NEXT-2)")
    ap.add_argument("--hbm-frac", type=float, default=-1.0, help="override the HBM-tier share of V (tier ablation)")
    ap.add_argument("--host-frac", type=float, default=-1.0, help="override the host-tier share of V (tier ablation)")
    ap.add_argument("--host-staged", type=float, default=1.0,
                    help="host tier: dynamic split between GPU zero-copy reads and host stager threads, with this "
                         "cap on the stagers' share of a batch's host rows (default 1.0 = no cap); 0 = pure zero-copy")
    ap.add_argument("--zero-copy", action="store_true", help="ablation: pure GPU zero-copy host tier (= --host-staged 0)")
    ap.add_argument("--stage-reserve", type=float, default=0.7,
                    help="HOST_STAGED: share of each batch's host-row chunks (from the list's end) the GPU leaves to "
                         "the stagers, waiting a bounded time before copying them itself (0 = pure dynamic split)")
    ap.add_argument("--stage-workers", type=int, default=0,
                    help="host stager threads per rank (HOST_STAGED); 0 = min(14, host cores / local ranks - 2) (14 of the GPU box's 16 cores measured best)")
    ap.add_argument("--ring-depth", type=int, default=256)
    ap.add_argument("--io-ctas", type=int, default=32, help="CTA budget of each IO kernel (PAPER.md:244)")
    ap.add_argument("--io-sync", action="store_true", help="ablation: GIDS-style coupled IO (one warp per request)")
    ap.add_argument("--hbm-replicated", action="store_true",
                    help="C5-rep ablation: every rank's HBM tier holds the same hottest rows (no peer rows)")
    ap.add_argument("--io-sms", type=int, default=0,
                    help="run the IO kernel on a green-context partition of this many SMs (SURVEY NEXT-3; 0 = none)")
    args = ap.parse_args()
    if args.zero_copy:
        args.host_staged = 0.0
    if args.stage_workers <= 0:   # 14 of a 16-core host measured best; per rank, the host's cores / ranks - 2
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
        cores = len(os.sched_getaffinity(0)) // max(1, local_world)
        args.stage_workers = max(2, min(14, cores - 2))

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg0 = workloads.CONFIGS[args.config]
    if args.hbm_frac >= 0 or args.host_frac >= 0:   # tier ablations
        import dataclasses
        cfg0 = dataclasses.replace(cfg0, hbm_frac=args.hbm_frac if args.hbm_frac >= 0 else cfg0.hbm_frac,
                                   host_frac=args.host_frac if args.host_frac >= 0 else cfg0.host_frac,
                                   name=f"{cfg0.name}-hbm{cfg0.hbm_frac if args.hbm_frac < 0 else args.hbm_frac:g}"
                                        f"-host{cfg0.host_frac if args.host_frac < 0 else args.host_frac:g}")
    workdir = os.environ.get("HELIOS_BENCH_DIR", "/tmp")
    s = args.scale if args.scale > 0 else pick_scale(cfg0, world, workdir)
    cfg = workloads.scaled(cfg0, s)

    if args.impl == "reference":
        return reference_arm(args, cfg, rank, world)

    import torch
    import torch.distributed as dist
    # HELIOS_BENCH_ONE_GPU=1: every rank on cuda:0 with gloo (exercises the N>1 path on one GPU;
    # not a scaling measurement).  Default: one rank per GPU over NCCL.
    one_gpu = os.environ.get("HELIOS_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    backend = "gloo" if one_gpu else "nccl"
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    def allreduce(t, op=None):
        if world == 1:
            return t
        op = op or dist.ReduceOp.SUM
        if backend == "gloo":
            c_ = t.cpu()
            dist.all_reduce(c_, op=op)
            t.copy_(c_)
        else:
            dist.all_reduce(t, op=op)
        return t
    from paper_2310_00837_b200 import helios as H
    from paper_2310_00837_b200 import dist as hdist

    # ---- inputs (rank 0 generates; shared through /dev/shm when N > 1) ----
    t_setup = time.time()
    shm = f"helios_bench_{os.getppid()}" if world > 1 else None
    tab_bytes = cfg.V * cfg.R
    file_cfg = has_file_tier(cfg)
    fdir = os.path.join(workdir, f"helios_bench_{os.getppid() if world > 1 else os.getpid()}")
    if rank == 0:
        if keeps_table(cfg):
            buf = host_buffer(tab_bytes, f"{shm}_feat" if shm else None, create=True)
            table = np.frombuffer(buf, dtype=np.float32).reshape(cfg.V, cfg.dim)
        else:
            table = None
        if file_cfg:
            os.makedirs(fdir, exist_ok=True)
        inp = workloads.make_inputs(cfg, table=table is not None, table_buffer=table, file=file_cfg, workdir=fdir)
        if world > 1:
            np.save(f"/dev/shm/{shm}_indptr.npy", inp.graph.indptr)
            np.save(f"/dev/shm/{shm}_indices.npy", inp.graph.indices)
    if world > 1:
        dist.barrier()
        if rank != 0:
            table = None
            if keeps_table(cfg):
                buf = host_buffer(tab_bytes, f"{shm}_feat", create=False)
                table = np.frombuffer(buf, dtype=np.float32).reshape(cfg.V, cfg.dim)
            gr = synth.Graph(cfg.V, np.load(f"/dev/shm/{shm}_indptr.npy", mmap_mode="r"),
                             np.load(f"/dev/shm/{shm}_indices.npy", mmap_mode="r"))
            train = synth.train_set(cfg.V, workloads.SEED, cfg.train_pct)
            path = os.path.join(fdir, f"features_{cfg.name}.bin") if file_cfg else None
            inp = workloads.Inputs(cfg, gr, table, path, 4096, (cfg.R + 511) // 512 * 512, train,
                                   synth.epoch_batches(train, cfg.B, 0, workloads.SEED))
    gen_s = time.time() - t_setup
    log(f"inputs {cfg.name}: V={cfg.V} E={inp.graph.E} dim={cfg.dim} gen {gen_s:.1f}s")

    t1 = time.time()
    g = H.helios_graph_load(inp.graph.indptr, inp.graph.indices, device=local,
                            flags=H.GRAPH_TOPO_HOST if args.topo_host else 0)
    full_batches = [b for b in inp.batches if len(b) == cfg.B]
    # presample: one epoch with presample keys, split over ranks, hotness all-reduced (NCCL)
    hot = torch.zeros(cfg.V, dtype=torch.int64, device="cuda")
    mine = [b for b in range(len(inp.batches)) if b % world == rank]
    pkeys = workloads.presample_keys(len(inp.batches))
    for b in mine:
        H.helios_presample(g, torch.as_tensor(inp.batches[b]).cuda(), cfg.B, cfg.fanouts, [pkeys[b]], hot)
    H.helios_graph_sync(g)
    allreduce(hot)
    presample_s = time.time() - t1
    Gd = 1 if args.hbm_replicated else world   # the directory's world size (C5-rep: replicated HBM tier)
    Hr, S = workloads.tier_rows(cfg, Gd)
    if cfg.hbm_frac + cfg.host_frac >= 1.0:
        S = max(0, cfg.V - Gd * Hr)
    else:
        S = max(0, min(S, cfg.V - Gd * Hr))
    t2 = time.time()
    fkw = dict(feature_path=inp.feature_path, header_bytes=inp.header, file_stride=inp.stride,
               io_rings=args.io_rings, ring_depth=args.ring_depth, io_ctas=args.io_ctas,
               io_sms=args.io_sms) if file_cfg else {}
    if args.host_staged > 0:
        fkw.update(stage_workers=args.stage_workers, stage_frac=args.host_staged,
                   stage_reserve=min(args.stage_reserve, args.host_staged))
    sflag = ((H.HOST_STAGED if args.host_staged > 0 else 0) | (H.IO_SYNC if args.io_sync else 0)
             | (H.HBM_REPLICATED if args.hbm_replicated else 0))
    if (args.host_alias and table is not None) or S == 0:
        c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=table, world_size=world, rank=rank,
                                 flags=(H.HOST_ALIAS if S else 0) | sflag, **fkw)
    elif world == 1:   # packed host tier in hot-rank order, pinned by the library
        c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=table, flags=sflag, **fkw)
    else:              # one packed host tier shared by all ranks (/dev/shm), filled by rank 0
        if rank == 0:  # creator first; the other ranks map the filled tier after the barrier
            tier_buf = host_buffer(S * cfg.R, f"{shm}_tier", create=True)
            tier = np.frombuffer(tier_buf, dtype=np.uint8)
            c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=table, world_size=world, rank=rank,
                                     host_tier=tier, flags=H.HOST_FILL | sflag, **fkw)
        dist.barrier()
        if rank != 0:
            tier_buf = host_buffer(S * cfg.R, f"{shm}_tier", create=False)
            tier = np.frombuffer(tier_buf, dtype=np.uint8)
            c = H.helios_cache_build(g, hot, cfg.R, Hr, S, host_table=table, world_size=world, rank=rank,
                                     host_tier=tier, flags=sflag, **fkw)
    if world > 1:
        hdist.attach_peers(H, c)
        dist.barrier()
    build_s = time.time() - t2
    log(f"graph load + presample {presample_s:.1f}s, cache build {build_s:.1f}s (H={Hr}/GPU, S={S})")

    # ---- timed loop: the execution plan (CUDA graphs, `depth` batches in flight) ----
    L = len(cfg.fanouts)
    keys = workloads.batch_keys(0, len(inp.batches))
    my_batches = [b for b in range(len(full_batches)) if b % world == rank]
    need = args.warmup + args.steps
    seq = [my_batches[i % len(my_batches)] for i in range(need)]
    seed_of = {b: torch.as_tensor(inp.batches[b]).cuda() for b in sorted(set(seq))}
    stream = torch.cuda.current_stream()
    depth = args.depth if args.depth > 0 else (24 if S > 0 else 16)   # profiles/r02/retune_l2_defaults.jsonl
    # gather kernels of this cache: fused lookup+gather when every row is in HBM, else the
    # lookup, the HBM part and (with a host tier) the host part in its own kernel
    direct = S == 0 and not file_cfg and os.environ.get("HELIOS_GATHER_DIRECT") != "0" and not os.environ.get("HELIOS_GATHER_BULK")
    split = S > 0 and os.environ.get("HELIOS_GATHER_SPLIT_HOST") != "0"
    pflags = ((H.PLAN_NO_GRAPH if args.no_graph else 0) | (H.PLAN_SERIAL_GATHER if args.serial_gather else 0)
              | (H.PLAN_INTRA_BATCH if args.intra else 0) | (H.PLAN_LINK_STREAM if args.link_stream else 0))
    G = args.group
    plan = H.helios_plan_create(g, c, cfg.B, cfg.fanouts, depth=depth, flags=pflags, group=G)
    P = plan.positions   # depth x G batch positions; a group's kernels launch once for its G batches

    for i in range(args.warmup):
        H.helios_plan_submit(plan, i % P, seed_of[seq[i]], keys[seq[i]], stream)
    for k in range(P):
        H.helios_plan_wait(plan, k, stream)
    H.helios_sync(c)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    staged0 = c.info().staged_rows
    torch.cuda.nvtx.range_push("timed")
    with ClockSampler(local) as clk:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        H.helios_plan_mark(plan, stream)
        # device timing events on every launch of the last depth*1000 (all of them by default): the
        # per-launch segments give the stage times and the union of the gather segments' intervals
        timed_from = max(0, args.steps - depth * 1000 * G)
        for i in range(args.steps):
            b = seq[args.warmup + i]
            H.helios_plan_submit(plan, i % P, seed_of[b], keys[b], stream, timing=(i >= timed_from))
        for k in range(P):
            H.helios_plan_wait(plan, k, stream)
        end.record(stream)
        torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    H.helios_sync(c)
    staged_timed = c.info().staged_rows - staged0
    total_ms = start.elapsed_time(end)
    sample_ms, gather_ms, link_ms, gather_iv, link_iv = [], [], [], [], []
    for k in range(0, P, G):   # group leaders: one timing record per group launch (the launching submit)
        n_k = sum(1 for i in range(k + G - 1, args.steps, P) if i >= timed_from)
        for back in range(n_k):
            tb = H.helios_plan_timing(plan, k, back)
            sample_ms.append(tb.sample_ms)
            gather_ms.append(tb.gather_ms)
            gather_iv.append((tb.t_gather, tb.t_end))
            if tb.link_ms >= 0:
                link_ms.append(tb.link_ms)
    n_timed = len(gather_iv) * G   # batches of the timed launches
    gather_busy_ms = interval_union(gather_iv)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    allreduce(t, dist.ReduceOp.MAX)
    if world > 1:
        dist.barrier()
    max_ms = float(t.item())
    if args.profile:
        print(json.dumps({"profile_run": True, "ms_per_step": max_ms / args.steps}), flush=True)
        return
    # per-batch row counts of the timed batches (deterministic; re-run untimed through slot 0)
    st = [0, 0, 0, 0]
    n_rows = 0
    blk0, _, stats0 = plan.outputs[0]
    acc = []   # sampling access counts of the first batches (end-to-end sector-granular roofline)
    for i in range(args.steps):
        b = seq[args.warmup + i]
        H.helios_plan_submit(plan, 0, seed_of[b], keys[b], stream)
        H.helios_plan_wait(plan, 0, stream)
        stream.synchronize()
        st = [x + int(y) for x, y in zip(st, stats0.cpu().tolist())]
        n_rows += int(blk0.level_counts[L].item())
        if i < 16:
            acc.append(sampling_accesses(blk0.to_host(), inp.graph.indptr, cfg.fanouts))
    H.helios_sync(c)

    # ---- e2e: through the public API with host buffers (host seeds in, counts + tier stats out) ----
    host_seeds = {b: np.ascontiguousarray(inp.batches[b]) for b in sorted(set(seq))}
    out_host = np.empty((P, L + 1 + 4), dtype=np.int64)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_e2e = time.perf_counter()
    for i in range(args.steps):
        b = seq[args.warmup + i]
        k = i % P
        if i >= P:   # the position's previous batch: its result must be on the host before reuse
            H.helios_plan_readback(plan, k, out_host[k])
        H.helios_plan_submit(plan, k, host_seeds[b], keys[b], stream, readback=True)
    for i in range(max(0, args.steps - P), args.steps):
        H.helios_plan_readback(plan, i % P, out_host[i % P])
    e2e_s = time.perf_counter() - t_e2e
    H.helios_sync(c)
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    allreduce(e2e_t, dist.ReduceOp.MAX)
    e2e_s = float(e2e_t.item())
    # ---- parity at full size: GPU batches vs the oracle, bit for bit (rank 0) ----
    parity = None
    cpu = None
    if rank == 0 and not args.profile:
        import oracle
        checked, ok = 0, True
        pb = sorted(set(seq))[: args.parity_batches]
        for j, b in enumerate(pb):   # the timed launch configuration: plan slots + CUDA graphs
            k = j % P
            H.helios_plan_submit(plan, k, seed_of[b], keys[b], stream)
            H.helios_plan_wait(plan, k, stream)
            H.helios_sync(c)
            blocks, feats, _ = plan.outputs[k]
            got = blocks.to_host()
            ob = oracle.sample(inp.graph.indptr, inp.graph.indices, inp.batches[b], cfg.fanouts, keys[b])
            ok &= np.array_equal(got["nodes"], ob.nodes)
            for h in range(L):
                ok &= np.array_equal(got["block_indptr"][h], ob.block_indptr[h])
                ok &= np.array_equal(got["block_indices"][h], ob.block_indices[h])
            ref = oracle.gather(ob.nodes, cfg.R, table=table, path=inp.feature_path, header=inp.header,
                                stride=inp.stride)
            ok &= np.array_equal(feats[: len(ob.nodes)].cpu().numpy(), ref)
            checked += 1
        parity = {"batches": checked, "bit_exact": bool(ok), "checks": "nodes, block CSR, feature bytes"}
        if not args.no_cpu_baseline:
            dir_host = None
            if file_cfg:   # CPU-managed cache: FILE-tier rows by pread, the rest from memory
                dir_host = H.device_view(c.info().dir, cfg.V, torch.int64).cpu().numpy()
            r = run_oracle_baseline(inp, keys, args.cpu_budget, dir_=dir_host)
            ncpu = len(os.sched_getaffinity(0))
            rP = run_oracle_baseline(inp, keys, args.cpu_budget, dir_=dir_host, threads=ncpu)
            cpu = {"value": round(r["value"], 4), "unit": "batches/s", "cores": 1, "kind": "oracle",
                   "sample": f"{r['batches']} batches of {cfg.name} (first of epoch 0), single-threaded C++ oracle "
                             f"sample+gather ({'FILE-tier rows by buffered pread, ' if file_cfg else ''}"
                             f"{'other rows from the canonical host table' if table is not None else 'rows by pread from the feature file'}), "
                             f"{r['seconds']:.1f}s; P-core leg: the same oracle on {ncpu} threads, one independent batch "
                             f"per thread at a time, {rP['batches']} batches in {rP['seconds']:.1f}s",
                   "feature_gbs": round(r["gbs"], 3), "cores_P": ncpu, "value_P": round(rP["value"], 4),
                   "feature_gbs_P": round(rP["gbs"], 3), "cpu_model": cpu_model()}

    # ---- roofline of the dominant kernel (lookup+gather, K3/K4) ----
    probe = link_probe = lists_alone = None
    if S > 0 and not args.profile:
        n_probe, reps = 1 << 18, 8
        # (1) independent ceiling: a loads-only microkernel that is not K4 (best of 4 in-flight depths)
        l_ms, l_depth = H.helios_cache_probe_link(c, n_probe, seed=11, reps=4)
        link_probe = {"Mrows_s": round(n_probe / l_ms / 1e3, 2), "gbs": round(n_probe * cfg.R / l_ms / 1e6, 2),
                      "how": f"helios_cache_probe_link: loads-only microkernel (not K4), {n_probe} uniformly random "
                             f"host-tier rows per launch, fresh rows every launch, best of 16 grid x loads-in-flight "
                             f"settings (best: ~{l_depth} rows in flight)"}
        # (2) K4's own host part on uniform random rows (the round-1 probe; kept for comparison)
        p_ms = H.helios_cache_probe_host(c, n_probe, seed=7, reps=reps)
        probe = {"Mrows_s": round(n_probe / p_ms / 1e3, 2), "gbs": round(n_probe * cfg.R / p_ms / 1e6, 2),
                 "how": f"helios_cache_probe_host: K4 host part alone, {n_probe} uniformly random host-tier rows per "
                        f"launch, fresh rows each of {reps} launches (no L2 reuse)"}
        # (3) the real lists alone: K3+K4 (helios_gather) on the first sampled batches of the run, one at
        # a time on an otherwise idle GPU (no concurrent sampling), device-timed
        blkA, featsA, statsA = plan.outputs[0]
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot_ms, tot_host, tot_rows = 0.0, 0, 0
        H.helios_gather(c, blkA.nodes, blkA.level_counts[L:L + 1], featsA, statsA, stream)  # workspace warm-up
        H.helios_sync(c)
        for i in range(min(8, args.steps)):
            b = seq[args.warmup + i]
            H.helios_plan_submit(plan, 0, seed_of[b], keys[b], stream)
            H.helios_plan_wait(plan, 0, stream)
            stream.synchronize()
            ev0.record(stream)
            H.helios_gather(c, blkA.nodes, blkA.level_counts[L:L + 1], featsA, statsA, stream)
            ev1.record(stream)
            ev1.synchronize()
            H.helios_sync(c)
            tot_ms += ev0.elapsed_time(ev1)
            stt = statsA.cpu().tolist()
            tot_host += stt[2]
            tot_rows += int(blkA.level_counts[L].item())
        lists_alone = {"Mrows_s_host": round(tot_host / tot_ms / 1e3, 2), "ms_per_batch": round(tot_ms / 8, 4),
                       "host_rows_per_batch": round(tot_host / 8, 1),
                       "how": "helios_gather (K3 + K4, host tier mode as configured) on 8 real sampled batches of the "
                              "run, one at a time on an idle GPU, CUDA events; host rows / gather time"}
    pk = measured_peaks()
    bw_hbm = float(pk.get("hbm_gbs", HBM_PEAK_FALLBACK))
    bw_pcie = pcie_h2d_peak(torch) if rank == 0 else 0.0
    bw_nvl = 770.0  # measured peer copy per direction (B200_PROFILING.md); 1 GPU runs have no peer rows
    R = cfg.R
    steps = args.steps
    n_local, n_peer, n_host, n_file = (x / steps for x in st)
    nL = n_rows / steps
    hbm_bytes = R * n_local + R * nL + 16 * nL         # tier read + output write + nodes/dir reads
    pcie_bytes = R * (n_host + n_file)
    nvl_bytes = R * n_peer
    stor_bytes = inp.stride * n_file if file_cfg else 0.0
    fpk = file_peak(inp.feature_path, inp.stride, inp.header, args.io_rings) if (file_cfg and rank == 0) else None
    bw_file = fpk["gbs"] if fpk else 1.0
    g_ms = statistics.mean(gather_ms)
    terms = {"hbm": hbm_bytes / bw_hbm, "pcie": pcie_bytes / max(bw_pcie, 1e-9), "nvlink": nvl_bytes / bw_nvl,
             "storage": stor_bytes / bw_file}
    t_roof_ms = sum(terms.values()) / 1e6
    alg_bytes = hbm_bytes + pcie_bytes + nvl_bytes + stor_bytes
    dominant = max(terms.items(), key=lambda x: x[1])[0]
    if plan.link and link_ms and not file_cfg:
        # dominant kernel = the host-row kernel on the link stream: its PCIe bytes per launch over
        # its own launch time (events on the link stream, one batch at a time by construction)
        l_ms = statistics.mean(link_ms)
        achieved = R * n_host / (l_ms * 1e6)
        roof = {"bound": "pcie", "kernel": "k_gather_lists<host part> (link stream)", "achieved": round(achieved, 2),
                "peak": round(bw_pcie, 2), "unit": "GB/s", "frac": round(achieved / bw_pcie, 4),
                "traffic": traffic_of(cfg.name + "/host"), "launch_ms": round(l_ms, 4),
                "note": "achieved = R*host_rows per launch / mean launch time (CUDA events on the link stream over the "
                        "timed region); peak = pinned H2D copy-engine bandwidth measured in this run; the platform's "
                        "random 512 B zero-copy ceiling is lower (DESIGN.md §6); tier sum form: t_roof_ms, frac_throughput"}
    else:
        # gathers of the `depth` slots overlap, so one launch's duration is shared with the others:
        # achieved = the timed launches' algorithmic bytes / the time at least one of them was running
        achieved = alg_bytes * n_timed / (gather_busy_ms * 1e6)
        peak = alg_bytes / (t_roof_ms * 1e6)
        kname = ("k_gather_direct (K3 fused into K4: every row in HBM)" if direct else
                 "k_lookup + k_gather_lists + k_gather_host (K3 + K4 HBM part + K4 host part)" if split else
                 "k_lookup + k_gather_lists (K3+K4)")
        roof = {"bound": dominant, "kernel": kname, "achieved": round(achieved, 2),
                "peak": round(peak, 2), "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic_of(cfg.name), "launch_ms": round(g_ms, 4),
                "busy_ms": round(gather_busy_ms, 3), "launches_timed": n_timed,
                "note": "achieved = algorithmic tier bytes (HBM tier read + output write + ids/dir, PCIe host rows, "
                        "NVLink peer rows, storage) of the timed launches / union of their execution intervals "
                        f"(CUDA events on the slot streams over the timed region; {P} batches in flight in {depth} "
                        f"groups of {G}, each group one launch of every kernel, so launches overlap); peak = the same bytes / T_roof, the tier sum form "
                        "sum(bytes_link / BW_link); frac_throughput = T_roof / ms_per_step"}
    roof.update({
        "peaks_used": {"hbm_gbs": bw_hbm, "hbm_src": "MEASURED_PEAKS.json" if pk else "fallback",
                       "pcie_gbs": round(bw_pcie, 2), "pcie_src": "pinned H2D copy measured in this run",
                       "nvlink_gbs": bw_nvl, "file_gbs": round(bw_file, 4) if fpk else None,
                       "file_src": f"tools/filebench random {inp.stride} B O_DIRECT={fpk['direct']} x{args.io_rings} threads" if fpk else None},
        "bytes_per_launch": {"hbm": round(hbm_bytes), "pcie": round(pcie_bytes), "nvlink": round(nvl_bytes),
                             "storage": round(stor_bytes)},
        "t_roof_ms": round(t_roof_ms, 4),
        "frac_throughput": round(t_roof_ms / (max_ms / steps), 4)})
    # end-to-end (sampling + lookup + gather) bound: streaming bytes at the HBM copy peak plus random
    # 32 B sectors at the random-sector rate measured live over this graph's CSR, plus the host link
    n_rs = 1 << 24
    sec_rate = n_rs / (H.helios_graph_probe_random(g, n_rs, reps=5) * 1e6) if not args.topo_host else None  # sectors/ns
    if acc and sec_rate:
        a_sec = statistics.mean(x["sectors"] for x in acc)
        a_str = statistics.mean(x["stream_bytes"] for x in acc) + hbm_bytes
        t_e2e = (a_str / bw_hbm + a_sec / sec_rate + pcie_bytes / max(bw_pcie, 1e-9) + nvl_bytes / bw_nvl
                 + stor_bytes / bw_file) / 1e6
        roof["end_to_end"] = {"random_sectors_per_batch": round(a_sec), "stream_bytes_per_batch": round(a_str),
                              "sector_rate_G_s": round(sec_rate, 2), "t_roof_ms": round(t_e2e, 4),
                              "frac": round(t_e2e / (max_ms / steps), 4),
                              "note": "whole step vs stream/BW_hbm + sectors/sector_rate + tier-link terms; sectors = "
                                      "per hop one per frontier row (indptr) + the expected distinct sectors holding its k "
                                      "sampled positions + one per node (directory), averaged over the first 16 timed "
                                      "batches (bench.sampling_accesses); sector_rate = helios_graph_probe_random "
                                      "(uniform 4 B loads over the CSR indices)"}
    if link_probe is not None and n_host > 0:
        got = n_host * (world * steps / (max_ms / 1e3)) / world / 1e6
        st_rows = staged_timed / steps if args.host_staged > 0 else 0.0
        zc = max(0.0, n_host - st_rows) * (steps / (max_ms / 1e3)) / 1e6  # GPU zero-copy rows (upper bound)
        roof["host_link"] = {"achieved_Mrows_s": round(got, 2), "random_row_ceiling": link_probe,
                             "frac_of_ceiling": round(got / link_probe["Mrows_s"], 4),
                             "zero_copy_Mrows_s": round(zc, 2),
                             "zero_copy_frac_of_ceiling": round(zc / link_probe["Mrows_s"], 4),
                             "k4_host_part_uniform_rows": probe, "real_lists_alone": lists_alone,
                             "cpu_staged_rows_per_batch": round(staged_timed / steps, 1) if args.host_staged > 0 else 0,
                             "note": "host-tier rows per second of the whole timed run (zero-copy and staged rows) vs "
                                     "the random zero-copy row ceiling measured by an independent loads-only kernel "
                                     "(DESIGN.md §6); the staged share can exceed the zero-copy ceiling because host "
                                     "threads stream it; zero_copy_* counts only the rows the stagers did not copy "
                                     "(a lower bound on the stagers' share, since a chunk both sides copy is counted "
                                     "as staged)"}
    value = world * steps / (max_ms / 1e3)
    e2e_val = world * steps / e2e_s
    # per group launch: the sampling chain (3L + 2 kernels), the gather kernels, the staged-tier publish;
    # per batch: the IO kernel + its finish (file tier), the link-stream host kernel (G = 1 only)
    gather_kernels = 1 if direct else (3 if split else 2)   # fused lookup+gather | lookup, HBM part, host part
    per_group = 3 * L + 2 + gather_kernels + (1 if (args.host_staged > 0 and S > 0) else 0)
    per_batch = (2 if c.info().file_rows > 0 else 0) + (1 if plan.link else 0)
    gpu_launches = per_group * ((steps + G - 1) // G) + per_batch * steps
    out = {
        "metric": "sampled+gathered mini-batches/sec (feature GB/s and tier-roofline fraction alongside)",
        "value": round(value, 3), "unit": "batches/s", "n_gpus": 1 if one_gpu else world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": round(max_ms / steps, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int64 ids / fp32 feature bytes (u8 copy)",
        "data": "synthetic (seeded R-MAT-marginal power-law graph, synth_feature rows; no datasets)",
        "config": {"workload": cfg.name, "desc": cfg.note, "V": cfg.V, "E": int(inp.graph.E), "dim": cfg.dim,
                   "file_tier": {"rows": int(c.info().file_rows), "direct_io": bool(c.info().direct_io),
                                 "io_rings": args.io_rings, "ring_depth": args.ring_depth, "io_ctas": args.io_ctas,
                                 "io_mode": "sync (GIDS-style ablation)" if args.io_sync else "decoupled submit/complete",
                                 "io_sms": int(c.info().io_sms) or "all (no partition)"}
                   if file_cfg else None,
                   "batch_per_rank": cfg.B, "fanouts": cfg.fanouts, "hbm_rows_per_gpu": Hr, "host_rows": S,
                   "scale": s, "parallelism": f"dp{world} (seeds split per rank, HBM tier "
                                              f"{'replicated' if args.hbm_replicated else 'sharded'})",
                   "host_tier": ("alias of canonical table (by id)" if args.host_alias else "packed, hot-rank order")
                   + (f"; dynamic split: GPU zero-copy from the front of each batch's host list, {args.stage_workers} "
                      f"host stager threads from its end (cap {args.host_staged:.0%}, last "
                      f"{min(args.stage_reserve, args.host_staged):.0%} reserved for the stagers)"
                      if args.host_staged > 0 else "; GPU zero-copy reads only (ablation)"),
                   "host_rows_kernel": ("combined (2 host warps per 8 in K4)" if os.environ.get("HELIOS_GATHER_SPLIT_HOST") == "0"
                                        else "split (own 64-thread kernel behind the HBM part)") if S > 0 else None,
                   "batches_in_flight": P, "plan_slots": depth, "batches_per_launch": G, "cuda_graphs": not args.no_graph, "serial_gather": bool(args.serial_gather),
                   "link_stream": bool(plan.link),
                   "table_home": {"0": "whole table"}.get(os.environ.get("HELIOS_TABLE_HOME", ""),
                                                         "adaptive (2^k >= 2.5 n_L of the slot's previous batch)"
                                                         if "HELIOS_TABLE_HOME" not in os.environ else
                                                         f"fixed {os.environ['HELIOS_TABLE_HOME']} slots"),
                   "gather_l2_policy": "evict_first (fused HBM-only gather)" if S == 0 and os.environ.get("HELIOS_GATHER_EVICT", "1") != "0"
                                       else "default",
                   "intra_batch_pipeline": bool(args.intra),
                   "topology": "pinned host, zero-copy (UVA)" if args.topo_host else "HBM",
                   "tiers": {"hbm_frac": cfg.hbm_frac, "host_frac": cfg.host_frac},
                   "l2": "inputs larger than L2 (CSR %.1f GB, feature table %.1f GB); no flush" % (
                       (inp.graph.E * 4 + cfg.V * 8) / 1e9, cfg.V * R / 1e9)},
        "feature_gbs": round(world * n_rows / steps * R * steps / (max_ms / 1e3) / 1e9, 2),
        "stage_ms": {"sample": round(statistics.mean(sample_ms), 4), "gather": round(g_ms, 4),
                     "link_host_kernel": round(statistics.mean(link_ms), 4) if link_ms else None,
                     "note": f"mean per launch ({G} batch(es) each), device events around the two graph segments of every timed launch ({len(gather_iv)}), {P} batches in flight"},
        "lookups_per_s": round(world * nL * steps / (max_ms / 1e3)),
        "rows_per_batch": {"n_L": round(nL, 1), "hbm_local": round(n_local, 1), "hbm_peer": round(n_peer, 1),
                           "host": round(n_host, 1), "file": round(n_file, 1)},
        "roofline": roof,
        "e2e": {"value": round(e2e_val, 3), "unit": "batches/s", "h2d_bytes_per_step": cfg.B * 8,
                "d2h_bytes_per_step": (L + 1 + 4) * 8},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "parity": parity,
        "setup_s": {"inputs": round(gen_s, 1), "load_presample": round(presample_s, 1), "cache_build": round(build_s, 1)},
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()   # no rank frees its HBM shard while another may still read it over NVLink
    plan.free()
    c.free()
    g.free()
    if file_cfg and rank == 0:
        import shutil
        shutil.rmtree(fdir, ignore_errors=True)
    if world > 1:
        dist.barrier()
        if rank == 0:
            for suf in ("_feat", "_tier", "_indptr.npy", "_indices.npy"):
                try:
                    os.unlink(f"/dev/shm/{shm}{suf}")
                except OSError:
                    pass
        dist.destroy_process_group()


def reference_arm(args, cfg, rank, world):
    """--impl reference: the oracle (the only reference this paper has) on the host cores."""
    if rank != 0:
        return
    import oracle
    t0 = time.time()
    file_cfg = has_file_tier(cfg)
    fdir = os.path.join(os.environ.get("HELIOS_BENCH_DIR", "/tmp"), f"helios_ref_{os.getpid()}")
    if file_cfg:
        os.makedirs(fdir, exist_ok=True)
    inp = workloads.make_inputs(cfg, table=keeps_table(cfg), file=file_cfg and not keeps_table(cfg), workdir=fdir)
    gen_s = time.time() - t0
    keys = workloads.batch_keys(0, len(inp.batches))
    full = [b for b in inp.batches if len(b) == cfg.B]
    L = len(cfg.fanouts)
    for i in range(args.warmup):
        ob = oracle.sample(inp.graph.indptr, inp.graph.indices, full[i % len(full)], cfg.fanouts, keys[i % len(full)])
        oracle.gather(ob.nodes, cfg.R, table=inp.table, path=inp.feature_path, header=inp.header, stride=inp.stride)
    t1 = time.perf_counter()
    rows = 0
    for i in range(args.steps):
        b = (args.warmup + i) % len(full)
        ob = oracle.sample(inp.graph.indptr, inp.graph.indices, full[b], cfg.fanouts, keys[b])
        oracle.gather(ob.nodes, cfg.R, table=inp.table, path=inp.feature_path, header=inp.header, stride=inp.stride)
        rows += len(ob.nodes)
    dt = time.perf_counter() - t1
    v = args.steps / dt
    if file_cfg:
        import shutil
        shutil.rmtree(fdir, ignore_errors=True)
    print(json.dumps({
        "impl": "reference", "metric": "sampled+gathered mini-batches/sec (feature GB/s and tier-roofline fraction alongside)",
        "value": round(v, 4), "unit": "batches/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3 / args.steps, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64 ids / fp32 feature bytes (u8 copy)", "data": "synthetic",
        "config": {"workload": cfg.name, "desc": cfg.note, "V": cfg.V, "E": int(inp.graph.E), "dim": cfg.dim,
                   "batch_per_rank": cfg.B, "fanouts": cfg.fanouts},
        "feature_gbs": round(rows * cfg.R / dt / 1e9, 3),
        "cpu_baseline": {"value": round(v, 4), "unit": "batches/s", "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} full batches of {cfg.name}, single-threaded C++ oracle",
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(v, 4), "unit": "batches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": {"inputs": round(gen_s, 1)},
    }), flush=True)


if __name__ == "__main__":
    main()
