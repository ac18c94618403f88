"""Thin ctypes binding of libhelios.so (C ABI v2, include/helios.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only turns torch tensors
into device pointers, torch streams into cudaStream_t handles, and statuses into exceptions.  There
is no CPU fallback: importing this module fails loudly when libhelios.so is missing.
Function names are the ABI's.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
# Plans run one stream per in-flight batch: ask for 32 hardware work queues (default 8) unless the
# caller chose otherwise; effective only if CUDA is not initialised yet in this process.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

_HERE = os.path.dirname(os.path.abspath(__file__))
# HELIOS_LIB=trace loads the traced build (device pipeline timeline, tools/trace_pipeline.py); HELIOS_LIB=<x>
# loads libhelios_<x>.so (same-box A/B of another build of the same ABI)
_LIB = os.environ.get("HELIOS_LIB")
SO_PATH = os.path.join(_HERE, f"libhelios_{_LIB}.so" if _LIB else "libhelios.so")
if not os.path.exists(SO_PATH):
    raise ImportError(f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(nvcc, sm_100a). There is no CPU fallback.")
_lib = ctypes.CDLL(SO_PATH)

MAX_HOPS = 8
MAX_RANKS = 64
STATUS = ["OK", "E_INVALID", "E_RANGE", "E_CAPACITY", "E_NOMEM", "E_CUDA", "E_IO", "E_TIMEOUT", "E_STATE"]
HOST_ALIAS, TABLE_MAPPED, NO_DIRECT_IO, IO_FAULT_AT = 0x1, 0x2, 0x4, 0x100
HOST_FILL, HOST_TIER_MAPPED, HOST_STAGED, IO_SYNC = 0x8, 0x10, 0x20, 0x40
HBM_REPLICATED = 0x200
PLAN_NO_GRAPH, PLAN_SERIAL_GATHER, PLAN_INTRA_BATCH, PLAN_LINK_STREAM, PLAN_TRACE = 0x1, 0x2, 0x4, 0x8, 0x10
SUBMIT_SEEDS_HOST, SUBMIT_TIMING, SUBMIT_READBACK, SUBMIT_FLUSH = 0x1, 0x2, 0x4, 0x8

i64, i32, u32, u64, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p


class helios_blocks(ctypes.Structure):
    _fields_ = [("nodes", vp), ("nodes_cap", i64), ("level_counts", vp), ("edge_counts", vp),
                ("block_indptr", vp * MAX_HOPS), ("indptr_cap", i64 * MAX_HOPS),
                ("block_indices", vp * MAX_HOPS), ("edges_cap", i64 * MAX_HOPS)]


class helios_cache_desc(ctypes.Structure):
    _fields_ = [("row_bytes", i32), ("world_size", i32), ("rank", i32), ("hbm_rows", i64), ("host_rows", i64),
                ("hotness", vp), ("host_table", vp), ("feature_path", ctypes.c_char_p), ("header_bytes", i64),
                ("file_stride", i64), ("io_rings", i32), ("ring_depth", i32), ("io_ctas", i32),
                ("io_fault_at", i32), ("flags", u32), ("host_tier", vp), ("stage_workers", i32),
                ("stage_frac", ctypes.c_float), ("stage_reserve", ctypes.c_float), ("io_sms", i32)]


class helios_plan_desc(ctypes.Structure):
    _fields_ = [("max_seeds", i64), ("L", i32), ("fanouts", i32 * MAX_HOPS), ("depth", i32), ("flags", u32),
                ("group", i32)]


class helios_batch_timing(ctypes.Structure):
    _fields_ = [("sample_ms", ctypes.c_float), ("gather_ms", ctypes.c_float), ("link_ms", ctypes.c_float),
                ("t_start", ctypes.c_float), ("t_gather", ctypes.c_float), ("t_end", ctypes.c_float)]


class helios_cache_info(ctypes.Structure):
    _fields_ = [("dir", vp), ("hbm_tier", vp), ("host_tier", vp), ("V", i64), ("hbm_rows", i64), ("host_rows", i64),
                ("file_rows", i64), ("row_bytes", i32), ("world_size", i32), ("rank", i32), ("peers_attached", i32),
                ("io_rings", i32), ("ring_depth", i32), ("direct_io", i32), ("io_reads", i64), ("staged_rows", i64), ("io_sms", i32)]


_sig = {
    "helios_abi_version": (ctypes.c_int, []),
    "helios_last_error": (ctypes.c_char_p, []),
    "helios_graph_load": (ctypes.c_int, [ctypes.c_int, i64, i64, vp, vp, u32, ctypes.POINTER(vp)]),
    "helios_graph_free": (None, [vp]),
    "helios_graph_info": (ctypes.c_int, [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_int)]),
    "helios_graph_device_csr": (ctypes.c_int, [vp, ctypes.POINTER(vp), ctypes.POINTER(vp)]),
    "helios_sample_bounds": (ctypes.c_int, [i64, vp, i32, i64, i64, ctypes.POINTER(i64), vp, vp]),
    "helios_sample": (ctypes.c_int, [vp, vp, i64, vp, i32, u64, ctypes.POINTER(helios_blocks), vp]),
    "helios_graph_probe_random": (ctypes.c_int, [vp, i64, i32, ctypes.POINTER(ctypes.c_float)]),
    "helios_graph_sync": (ctypes.c_int, [vp, vp]),
    "helios_presample": (ctypes.c_int, [vp, vp, i64, i32, vp, i32, vp, vp, vp]),
    "helios_cache_build": (ctypes.c_int, [vp, ctypes.POINTER(helios_cache_desc), ctypes.POINTER(vp)]),
    "helios_cache_free": (None, [vp]),
    "helios_cache_query": (ctypes.c_int, [vp, ctypes.POINTER(helios_cache_info)]),
    "helios_cache_export": (ctypes.c_int, [vp, vp, ctypes.POINTER(ctypes.c_size_t)]),
    "helios_cache_attach_peers": (ctypes.c_int, [vp, vp, ctypes.c_size_t]),
    "helios_gather": (ctypes.c_int, [vp, vp, vp, i64, vp, vp, vp]),
    "helios_cache_probe_host": (ctypes.c_int, [vp, i64, u64, i32, ctypes.POINTER(ctypes.c_float)]),
    "helios_cache_probe_link": (ctypes.c_int, [vp, i64, u64, i32, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32)]),
    "helios_batch_prepare": (ctypes.c_int, [vp, vp, vp, i64, vp, i32, u64, ctypes.POINTER(helios_blocks), vp, vp, vp]),
    "helios_sync": (ctypes.c_int, [vp, vp]),
    "helios_plan_create": (ctypes.c_int, [vp, vp, ctypes.POINTER(helios_plan_desc), ctypes.POINTER(vp)]),
    "helios_plan_free": (None, [vp]),
    "helios_plan_outputs": (ctypes.c_int, [vp, i32, ctypes.POINTER(helios_blocks), ctypes.POINTER(vp),
                                           ctypes.POINTER(vp)]),
    "helios_plan_submit": (ctypes.c_int, [vp, i32, vp, i64, u64, u32, vp]),
    "helios_plan_readback": (ctypes.c_int, [vp, i32, vp]),
    "helios_plan_wait": (ctypes.c_int, [vp, i32, vp]),
    "helios_plan_timing": (ctypes.c_int, [vp, i32, i32, ctypes.POINTER(helios_batch_timing)]),
    "helios_plan_mark": (ctypes.c_int, [vp, vp]),
    "helios_plan_trace": (ctypes.c_int, [vp, i32, i32, vp, i32, ctypes.POINTER(i32)]),
}
for _n, (_r, _a) in _sig.items():
    _f = getattr(_lib, _n)
    _f.restype = _r
    _f.argtypes = _a

ABI_SYMBOLS = tuple(_sig)


class HeliosError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        self.name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        detail = (_lib.helios_last_error() or b"").decode(errors="replace")
        super().__init__(f"{where}: HELIOS_{self.name}: {detail}")


def _check(st: int, where: str) -> None:
    if st != 0:
        raise HeliosError(st, where)


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return int(t)


def _stream(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _device_ids(t: torch.Tensor, stream) -> torch.Tensor:
    """int64, contiguous device ids for an enqueue-only call.  A converted copy is a temporary of the
    current torch stream: when the call enqueues on another stream, the copy is recorded on that
    stream so the caching allocator does not reuse its memory before the library's kernels read it."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("device ids must be a CUDA tensor")
    if t.dtype == torch.int64 and t.is_contiguous():
        return t
    c = t.to(torch.int64).contiguous()
    s = _stream(stream)
    if s != torch.cuda.current_stream().cuda_stream:
        c.record_stream(torch.cuda.ExternalStream(s))
    return c


def helios_abi_version() -> int:
    return _lib.helios_abi_version()


# ---- graph ---------------------------------------------------------------------------------------

class Graph:
    def __init__(self, handle: int, V: int, E: int, device: int):
        self.handle, self.V, self.E, self.device = handle, V, E, device

    def free(self):
        if self.handle:
            _lib.helios_graph_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


GRAPH_TOPO_HOST = 0x1


def helios_graph_load(indptr: np.ndarray, indices: np.ndarray, device: int = 0, flags: int = 0) -> Graph:
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    V, E = len(indptr) - 1, len(indices)
    h = vp()
    _check(_lib.helios_graph_load(device, V, E, _ptr(indptr), _ptr(indices) if E else None, flags, ctypes.byref(h)),
           "helios_graph_load")
    return Graph(h.value, V, E, device)


def helios_graph_device_csr(g: Graph) -> tuple[int, int]:
    a, b = vp(), vp()
    _check(_lib.helios_graph_device_csr(g.handle, ctypes.byref(a), ctypes.byref(b)), "helios_graph_device_csr")
    return a.value, b.value


def helios_sample_bounds(n_seeds: int, fanouts, V: int, E: int) -> tuple[int, list[int], list[int]]:
    fan = np.ascontiguousarray(fanouts, dtype=np.int32)
    L = len(fan)
    lvl = np.zeros(L + 1, dtype=np.int64)
    edg = np.zeros(max(L, 1), dtype=np.int64)
    mx = i64()
    _check(_lib.helios_sample_bounds(n_seeds, _ptr(fan), L, V, E, ctypes.byref(mx), _ptr(lvl), _ptr(edg)),
           "helios_sample_bounds")
    return mx.value, lvl.tolist(), edg[:L].tolist()


@dataclass
class Blocks:
    """Caller-owned device output buffers of one mini-batch, sized by helios_sample_bounds."""
    nodes: torch.Tensor
    level_counts: torch.Tensor
    edge_counts: torch.Tensor
    block_indptr: list
    block_indices: list
    fanouts: list

    @staticmethod
    def allocate(n_seeds: int, fanouts, V: int, E: int, device=0) -> "Blocks":
        mx, lvl, edg = helios_sample_bounds(n_seeds, fanouts, V, E)
        dev = torch.device("cuda", device) if isinstance(device, int) else device
        return Blocks(nodes=torch.empty(max(mx, 1), dtype=torch.int64, device=dev),
                      level_counts=torch.zeros(len(fanouts) + 1, dtype=torch.int64, device=dev),
                      edge_counts=torch.zeros(MAX_HOPS, dtype=torch.int64, device=dev),
                      block_indptr=[torch.empty(lvl[h] + 1, dtype=torch.int32, device=dev) for h in range(len(fanouts))],
                      block_indices=[torch.empty(max(edg[h], 1), dtype=torch.int32, device=dev)
                                     for h in range(len(fanouts))],
                      fanouts=list(fanouts))

    def struct(self) -> helios_blocks:
        s = helios_blocks()
        s.nodes = self.nodes.data_ptr()
        s.nodes_cap = self.nodes.numel()
        s.level_counts = self.level_counts.data_ptr()
        s.edge_counts = self.edge_counts.data_ptr()
        for h in range(len(self.fanouts)):
            s.block_indptr[h] = self.block_indptr[h].data_ptr()
            s.indptr_cap[h] = self.block_indptr[h].numel()
            s.block_indices[h] = self.block_indices[h].data_ptr()
            s.edges_cap[h] = self.block_indices[h].numel()
        return s

    def to_host(self) -> dict:
        """Copies the batch back (synchronises): nodes, level_counts, edge_counts, per-hop CSR."""
        L = len(self.fanouts)
        lc = self.level_counts.cpu().numpy()
        ec = self.edge_counts[:L].cpu().numpy()
        return {"nodes": self.nodes[: lc[L]].cpu().numpy(), "level_counts": lc, "edge_counts": ec,
                "block_indptr": [self.block_indptr[h][: lc[h] + 1].cpu().numpy() for h in range(L)],
                "block_indices": [self.block_indices[h][: ec[h]].cpu().numpy() for h in range(L)]}


def helios_sample(g: Graph, seeds: torch.Tensor, fanouts, key: int, out: Blocks, stream=None) -> None:
    fan = np.ascontiguousarray(fanouts, dtype=np.int32)
    seeds = _device_ids(seeds, stream)
    s = out.struct()
    _check(_lib.helios_sample(g.handle, _ptr(seeds), seeds.numel(), _ptr(fan), len(fan), key & (2**64 - 1),
                              ctypes.byref(s), _stream(stream)), "helios_sample")


def helios_graph_probe_random(g: Graph, n_reads: int, reps: int = 5) -> float:
    """Mean ms of n_reads uniformly random 4 B loads over the CSR indices (random-sector ceiling)."""
    ms = ctypes.c_float()
    _check(_lib.helios_graph_probe_random(g.handle, n_reads, reps, ctypes.byref(ms)), "helios_graph_probe_random")
    return ms.value


def helios_graph_sync(g: Graph, stream=None) -> None:
    _check(_lib.helios_graph_sync(g.handle, _stream(stream)), "helios_graph_sync")


def helios_presample(g: Graph, seeds: torch.Tensor, batch: int, fanouts, keys, hotness: torch.Tensor,
                     stream=None) -> None:
    fan = np.ascontiguousarray(fanouts, dtype=np.int32)
    ks = np.ascontiguousarray([k & (2**64 - 1) for k in keys], dtype=np.uint64)
    seeds = _device_ids(seeds, stream)
    if hotness.dtype not in (torch.int64, torch.uint64) or not hotness.is_contiguous() or not hotness.is_cuda:
        raise TypeError("hotness must be a contiguous 64-bit CUDA tensor [V] (accumulated in place)")
    _check(_lib.helios_presample(g.handle, _ptr(seeds), seeds.numel(), batch, _ptr(fan), len(fan), _ptr(ks),
                                 _ptr(hotness), _stream(stream)), "helios_presample")


# ---- cache ---------------------------------------------------------------------------------------

class Cache:
    def __init__(self, handle: int, graph: Graph, keepalive):
        self.handle, self.graph, self._keep = handle, graph, keepalive

    def info(self) -> helios_cache_info:
        inf = helios_cache_info()
        _check(_lib.helios_cache_query(self.handle, ctypes.byref(inf)), "helios_cache_query")
        return inf

    def free(self):
        if self.handle:
            _lib.helios_cache_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def helios_cache_build(g: Graph, hotness: torch.Tensor, row_bytes: int, hbm_rows: int, host_rows: int,
                       host_table: np.ndarray | None = None, feature_path: str | None = None, header_bytes: int = 0,
                       file_stride: int = 0, world_size: int = 1, rank: int = 0, io_rings: int = 4,
                       ring_depth: int = 256, io_ctas: int = 32, flags: int = 0, io_fault_at: int = 0,
                       host_tier=None, stage_workers: int = 0, stage_frac: float = 0.0,
                       stage_reserve: float = 0.0, io_sms: int = 0) -> Cache:
    d = helios_cache_desc()
    d.row_bytes, d.world_size, d.rank = row_bytes, world_size, rank
    d.hbm_rows, d.host_rows = hbm_rows, host_rows
    d.hotness = hotness.data_ptr()
    d.host_table = _ptr(host_table)
    path = feature_path.encode() if feature_path else None
    d.feature_path = path
    d.header_bytes, d.file_stride = header_bytes, file_stride
    d.io_rings, d.ring_depth, d.io_ctas, d.io_fault_at, d.flags = io_rings, ring_depth, io_ctas, io_fault_at, flags
    d.host_tier = _ptr(host_tier)
    d.stage_workers, d.stage_frac, d.stage_reserve = stage_workers, stage_frac, stage_reserve
    d.io_sms = io_sms
    h = vp()
    _check(_lib.helios_cache_build(g.handle, ctypes.byref(d), ctypes.byref(h)), "helios_cache_build")
    return Cache(h.value, g, (host_table, path, host_tier))


def helios_cache_export(c: Cache) -> bytes:
    n = ctypes.c_size_t(0)
    _check(_lib.helios_cache_export(c.handle, None, ctypes.byref(n)), "helios_cache_export")
    buf = ctypes.create_string_buffer(n.value)
    _check(_lib.helios_cache_export(c.handle, buf, ctypes.byref(n)), "helios_cache_export")
    return buf.raw[: n.value]


def helios_cache_attach_peers(c: Cache, blobs: list[bytes]) -> None:
    size = len(blobs[0])
    assert all(len(b) == size for b in blobs)
    buf = ctypes.create_string_buffer(b"".join(blobs), size * len(blobs))
    _check(_lib.helios_cache_attach_peers(c.handle, buf, size), "helios_cache_attach_peers")


def helios_gather(c: Cache, nodes: torch.Tensor, n_nodes: torch.Tensor, out: torch.Tensor,
                  stats: torch.Tensor | None = None, stream=None) -> None:
    nodes = _device_ids(nodes, stream)
    _check(_lib.helios_gather(c.handle, _ptr(nodes), _ptr(n_nodes), nodes.numel(), _ptr(out), _ptr(stats),
                              _stream(stream)), "helios_gather")


def helios_batch_prepare(g: Graph, c: Cache, seeds: torch.Tensor, fanouts, key: int, out: Blocks,
                         features: torch.Tensor, stats: torch.Tensor | None = None, stream=None) -> None:
    fan = np.ascontiguousarray(fanouts, dtype=np.int32)
    seeds = _device_ids(seeds, stream)
    s = out.struct()
    _check(_lib.helios_batch_prepare(g.handle, c.handle, _ptr(seeds), seeds.numel(), _ptr(fan), len(fan),
                                     key & (2**64 - 1), ctypes.byref(s), _ptr(features), _ptr(stats),
                                     _stream(stream)), "helios_batch_prepare")


def helios_cache_probe_host(c: Cache, n_rows: int, seed: int = 1, reps: int = 5) -> float:
    """Mean ms of K4's host part over n_rows uniformly random host-tier rows (fresh each rep)."""
    ms = ctypes.c_float()
    _check(_lib.helios_cache_probe_host(c.handle, n_rows, seed & (2**64 - 1), reps, ctypes.byref(ms)),
           "helios_cache_probe_host")
    return ms.value


def helios_cache_probe_link(c: Cache, n_rows: int, seed: int = 1, reps: int = 3) -> tuple[float, int]:
    """(best mean ms, rows in flight of that setting) of a loads-only random-row microkernel (not K4)
    over n_rows uniformly random host-tier rows, swept over grid size x loads in flight: the host
    link's random-row ceiling."""
    ms, d = ctypes.c_float(), i32()
    _check(_lib.helios_cache_probe_link(c.handle, n_rows, seed & (2**64 - 1), reps, ctypes.byref(ms), ctypes.byref(d)),
           "helios_cache_probe_link")
    return ms.value, d.value


def helios_sync(c: Cache, stream=None) -> None:
    _check(_lib.helios_sync(c.handle, _stream(stream)), "helios_sync")


def new_stats(device=0) -> torch.Tensor:
    """Device helios_gather_stats: int64[4] = rows_hbm_local, rows_hbm_peer, rows_host, rows_file."""
    return torch.zeros(4, dtype=torch.int64, device=torch.device("cuda", device) if isinstance(device, int) else device)


class _CudaArray:
    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False), "version": 3}


def device_view(ptr: int, n: int, dtype=torch.int64) -> torch.Tensor:
    """Zero-copy torch view of a library-owned device array (e.g. helios_cache_info.dir)."""
    typestr = {torch.int64: "<i8", torch.int32: "<i4", torch.uint8: "|u1", torch.float32: "<f4"}[dtype]
    return torch.as_tensor(_CudaArray(ptr, n, typestr), device="cuda")


# ---- execution plan ------------------------------------------------------------------------------

class Plan:
    """A helios_plan: `depth` in-flight batch slots of `group` batches each, each slot replaying a CUDA
    graph of its whole group.  `positions` = depth * group; every plan call takes a position.
    Position outputs are plan-owned device buffers exposed as zero-copy torch views."""

    def __init__(self, handle: int, graph: Graph, cache: Cache | None, B: int, fanouts, depth: int, group: int = 1):
        self.handle, self.graph, self.cache, self.B, self.fanouts, self.depth = handle, graph, cache, B, list(fanouts), depth
        self.group = group
        self.positions = depth * group
        # device seeds of each position's last submit: kept referenced until that position is reused, so
        # PyTorch's caching allocator cannot hand the memory out while the plan may still read it
        self._seeds_ref = [None] * self.positions
        L = len(self.fanouts)
        self.outputs = []
        for k in range(self.positions):
            blk, fp, sp = helios_blocks(), vp(), vp()
            _check(_lib.helios_plan_outputs(handle, k, ctypes.byref(blk), ctypes.byref(fp), ctypes.byref(sp)),
                   "helios_plan_outputs")
            b = Blocks(nodes=device_view(blk.nodes, blk.nodes_cap, torch.int64),
                       level_counts=device_view(blk.level_counts, L + 1, torch.int64),
                       edge_counts=device_view(blk.edge_counts, MAX_HOPS, torch.int64),
                       block_indptr=[device_view(blk.block_indptr[h], blk.indptr_cap[h], torch.int32) for h in range(L)],
                       block_indices=[device_view(blk.block_indices[h], max(1, blk.edges_cap[h]), torch.int32)
                                      for h in range(L)],
                       fanouts=self.fanouts)
            feats = stats = None
            if cache is not None:
                R = cache.info().row_bytes
                feats = device_view(fp.value, blk.nodes_cap * R, torch.uint8).view(blk.nodes_cap, R)
                stats = device_view(sp.value, 4, torch.int64)
            self.outputs.append((b, feats, stats))

    def free(self):
        if self.handle:
            _lib.helios_plan_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def helios_plan_create(g: Graph, c: Cache | None, B: int, fanouts, depth: int = 2, flags: int = 0,
                       group: int = 1) -> Plan:
    d = helios_plan_desc()
    d.max_seeds, d.L, d.depth, d.flags, d.group = B, len(fanouts), depth, flags, group
    for h, f in enumerate(fanouts):
        d.fanouts[h] = f
    h = vp()
    _check(_lib.helios_plan_create(g.handle, c.handle if c is not None else None, ctypes.byref(d), ctypes.byref(h)),
           "helios_plan_create")
    p = Plan(h.value, g, c, B, fanouts, depth, group)
    # host rows go through the plan's link stream (see helios.h, HELIOS_PLAN_LINK_STREAM)
    p.link = (c is not None and c.info().host_rows > 0 and bool(flags & PLAN_LINK_STREAM)
              and not flags & (PLAN_SERIAL_GATHER | PLAN_INTRA_BATCH))
    return p


def helios_plan_submit(p: Plan, slot: int, seeds, key: int, stream=None, timing: bool = False,
                       readback: bool = False, flush: bool = False) -> None:
    if isinstance(seeds, torch.Tensor) and seeds.is_cuda and seeds.dtype == torch.int64 and seeds.is_contiguous():
        # the plan reads them later on its slot stream (helios.h, helios_plan_submit): the binding keeps a
        # reference until the position's next submit, so they stay allocated while the batch can run
        ptr, n, fl, keep = seeds.data_ptr(), seeds.numel(), 0, seeds
    else:
        # host seeds, or device seeds needing a conversion: copied into the submit's parameter block
        # (no temporary device buffer whose lifetime the plan would have to track)
        if isinstance(seeds, torch.Tensor):
            seeds = seeds.detach().to("cpu", torch.int64).numpy()
        arr = np.ascontiguousarray(seeds, dtype=np.int64)
        ptr, n, fl, keep = _ptr(arr), len(arr), SUBMIT_SEEDS_HOST, None
    if timing:
        fl |= SUBMIT_TIMING
    if readback:
        fl |= SUBMIT_READBACK
    if flush:
        fl |= SUBMIT_FLUSH
    _check(_lib.helios_plan_submit(p.handle, slot, ptr, n, key & (2**64 - 1), fl, _stream(stream)),
           "helios_plan_submit")
    p._seeds_ref[slot] = keep


def helios_plan_readback(p: Plan, slot: int, out: np.ndarray | None = None) -> np.ndarray:
    """Blocks for slot's last batch (submitted with readback=True): int64[L + 1 + 4] = level counts,
    then rows_hbm_local, rows_hbm_peer, rows_host, rows_file."""
    if out is None:
        out = np.empty(len(p.fanouts) + 5, dtype=np.int64)
    _check(_lib.helios_plan_readback(p.handle, slot, _ptr(out)), "helios_plan_readback")
    return out


def helios_plan_wait(p: Plan, slot: int, stream=None) -> None:
    _check(_lib.helios_plan_wait(p.handle, slot, _stream(stream)), "helios_plan_wait")


def helios_plan_timing(p: Plan, slot: int, back: int = 0) -> helios_batch_timing:
    """Device timing of slot's timed batch `back` timed submissions ago (0 = last): sample_ms,
    gather_ms, link_ms (-1 without a link stream) and t_start / t_gather / t_end in ms since the last
    helios_plan_mark (-1 if never marked)."""
    t = helios_batch_timing()
    _check(_lib.helios_plan_timing(p.handle, slot, back, ctypes.byref(t)), "helios_plan_timing")
    return t


def helios_plan_trace(p: Plan, slot: int, back: int = 0) -> np.ndarray:
    """Per-kernel device timeline (ns, %globaltimer) of a traced batch: uint64[3L + 4, 2] of
    (first warp start, last warp end); rows 3h..3h+2 = count scan / fill / assign of hop h, then
    relabel, table clear, lookup, gather (0 = did not run).  Plan created with PLAN_TRACE."""
    K = 3 * len(p.fanouts) + 4
    out = np.zeros(2 * K, dtype=np.uint64)
    n = i32()
    _check(_lib.helios_plan_trace(p.handle, slot, back, _ptr(out), 2 * K, ctypes.byref(n)), "helios_plan_trace")
    return out.reshape(K, 2)


def helios_plan_mark(p: Plan, stream=None) -> None:
    _check(_lib.helios_plan_mark(p.handle, _stream(stream)), "helios_plan_mark")
