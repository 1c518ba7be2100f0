"""Multi-GPU sharding of a chunk batch: one process per GPU.

Chunks are independent (pipeline.py:358-367), so the data path
has no collective: rank r compresses a contiguous block of chunks on its own
GPU.  The one exchange is the final size all-gather (int64 per chunk) from
which every rank derives its span of the container; every rank writes its
records + payloads into one shared host segment (distributed.py; SURVEY.md
§8(e)).  Over NVLink/NVSwitch the all-gather is a few KB; with the gloo
backend the same code runs on CPU for the tests.
"""

from __future__ import annotations

import numpy as np

from .container import HEADER, RECORD


def shard_bounds(nchunks: int, world: int, rank: int) -> tuple:
    """Contiguous block [lo, hi) of chunk indices owned by ``rank``; the first
    ``nchunks % world`` ranks take one extra chunk."""
    base, extra = divmod(nchunks, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def exchange_sizes(local_sizes: np.ndarray, nchunks: int, group=None) -> np.ndarray:
    """All-gather per-chunk payload sizes (the only collective of the path)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    width = -(-nchunks // world) + 1
    buf = torch.full((width,), -1, dtype=torch.int64, device=dev)
    buf[: len(local_sizes)] = torch.as_tensor(np.asarray(local_sizes, np.int64), device=dev)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    sizes = []
    for r in range(world):
        lo, hi = shard_bounds(nchunks, world, r)
        sizes.append(out[r][: hi - lo].cpu().numpy())
    return np.concatenate(sizes) if sizes else np.zeros(0, np.int64)


def container_offsets(all_sizes: np.ndarray) -> np.ndarray:
    """Byte offset of each chunk's record in the container (42 B header,
    then 25 B record + payload per chunk)."""
    sizes = np.asarray(all_sizes, np.int64)
    rec = RECORD.size
    starts = np.zeros(len(sizes), np.int64)
    if len(sizes):
        starts[1:] = np.cumsum(sizes[:-1] + rec)
    return HEADER.size + starts


def compress_sharded(grid, params, compress_records=None, group=None):
    """Compress a GridArray with its (default-chunked) slices split across the
    ranks of ``group``: :func:`distributed.compress_shard` on this rank's
    block.  ``compress_records(stack) -> (records[RECORD_DTYPE], payload
    uint8, offsets)`` replaces the device coder (the CPU oracle in the
    multi-process tests); None = the GPU path.  Returns the container bytes
    on rank 0 and None elsewhere."""
    import torch.distributed as dist

    from .distributed import compress_shard
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    t, p, h, w = grid.dims
    lo, hi = shard_bounds(t * p, world, rank)
    stack = grid.data.reshape(t * p, h, w)[lo:hi]
    return compress_shard(stack, grid.dims, params.epsilon_rel, params.q, group=group,
                          coder=compress_records)
