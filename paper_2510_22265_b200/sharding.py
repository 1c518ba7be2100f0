"""Multi-GPU sharding of a chunk batch: one process per GPU.

Chunks are independent (pipeline.py:358-367), so the data path
has no collective: rank r compresses a contiguous block of chunks on its own
GPU.  The one exchange is the final size all-gather (int64 per chunk) from
which every rank derives its payload's offset in the container; the payload
bytes are then gathered to rank 0, which writes the container (SURVEY.md
§8(e)).  Over NVLink/NVSwitch the all-gather is a few KB; with the gloo
backend the same code runs on CPU for the tests.
"""

from __future__ import annotations

import numpy as np

from .container import HEADER, RECORD, RECORD_DTYPE, assemble


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


def compress_sharded(grid, params, compress_records, group=None):
    """Compress a GridArray with its (default-chunked) slices split across the
    ranks of ``group``.  ``compress_records(stack) -> (records[RECORD_DTYPE],
    payload uint8, offsets)`` is the per-rank batch compressor (the GPU path
    in production, the CPU oracle in tests).  Returns the container bytes on
    rank 0 and None elsewhere."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    t, p, h, w = grid.dims
    stack = grid.data.reshape(t * p, h, w)
    n = stack.shape[0]
    lo, hi = shard_bounds(n, world, rank)
    recs, payload, offs = compress_records(stack[lo:hi])
    local_sizes = (recs["base_len"].astype(np.int64) + recs["resid_len"].astype(np.int64))
    exchange_sizes(local_sizes, n, group)  # every rank learns the layout
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((recs.tobytes(), bytes(payload.tobytes()), offs.tolist()), gathered,
                       dst=0, group=group)
    if rank != 0:
        return None
    all_recs, parts, all_offs, base = [], [], [], 0
    for rb, pb, ob in gathered:
        r = np.frombuffer(rb, dtype=RECORD_DTYPE)
        all_recs.append(r)
        all_offs.extend(o + base for o in ob)
        parts.append(pb)
        base += len(pb)
    records = np.concatenate(all_recs) if all_recs else np.zeros(0, RECORD_DTYPE)
    payload = np.frombuffer(b"".join(parts), np.uint8)
    return assemble(grid.dims, grid.chunk_shape, records, payload, np.asarray(all_offs, np.int64))
