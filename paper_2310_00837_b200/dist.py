"""Multi-GPU plumbing for the Helios path — setup only, no per-batch collective.

* Seeds are split per rank: rank r takes batches b = r (mod N), each with its own key (weak scaling).
* The HBM tier is sharded round-robin by hot rank (the library's directory owner bits); peer rows
  are read by the gather kernel directly over NVLink through CUDA IPC-mapped peer shards.
* Collectives (torch.distributed, NCCL on GPUs / gloo in CPU tests), both at setup:
    1. all_reduce(SUM) of the hotness vector after each rank presampled its share of the batches;
    2. all_gather of each rank's helios_cache_export blob, then helios_cache_attach_peers.
* Host inputs shared by all ranks of a node live in /dev/shm mappings (one copy).
"""
from __future__ import annotations

import mmap
import os

import numpy as np


def rank_batches(n_batches: int, rank: int, world: int) -> list[int]:
    """Batches of this rank: b = rank (mod world)."""
    return list(range(rank, n_batches, world))


def allreduce_hotness(hot, group=None):
    """Sum the per-rank presample hotness vectors in place (hot[v] = # presample batches with v in N_L)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hot, op=dist.ReduceOp.SUM, group=group)
    return hot


def exchange_blobs(blob: bytes, group=None) -> list[bytes]:
    """All-gather of the per-rank cache export blobs (rank order)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [blob]
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


def attach_peers(H, cache, group=None) -> None:
    """Export this rank's HBM shard, all-gather the blobs and attach every peer's shard."""
    blobs = exchange_blobs(H.helios_cache_export(cache), group)
    if len(blobs) > 1:
        H.helios_cache_attach_peers(cache, blobs)


def shared_buffer(name: str, nbytes: int, create: bool) -> mmap.mmap:
    """A /dev/shm mapping shared by the ranks of one node (MAP_SHARED, transparent huge pages hint)."""
    path = f"/dev/shm/{name}"
    if create:
        fd = os.open(path, os.O_CREAT | os.O_RDWR | os.O_TRUNC, 0o600)
        os.ftruncate(fd, max(nbytes, 1))
    else:
        fd = os.open(path, os.O_RDWR)
    try:
        m = mmap.mmap(fd, max(nbytes, 1), flags=mmap.MAP_SHARED)
    finally:
        os.close(fd)
    try:
        m.madvise(mmap.MADV_HUGEPAGE)
    except (AttributeError, OSError):
        pass
    return m


def shared_array(name: str, shape, dtype, create: bool) -> tuple[np.ndarray, mmap.mmap]:
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) * dtype.itemsize
    m = shared_buffer(name, n, create)
    return np.frombuffer(m, dtype=dtype, count=int(np.prod(shape))).reshape(shape), m


def unlink_shared(name: str) -> None:
    try:
        os.unlink(f"/dev/shm/{name}")
    except OSError:
        pass
