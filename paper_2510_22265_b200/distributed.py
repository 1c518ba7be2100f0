"""Multi-GPU public API: one process per GPU on one node (torchrun).

The reference compresses chunks in a serial loop (pipeline.py:358-367) and
allows them to be processed concurrently; chunks share no
state, so the multi-GPU path shards them and has no collective on the data
path:

* rank r compresses the contiguous block ``sharding.shard_bounds(n, world,
  r)`` of the default chunks (one 2D slice per (t, p)) on its own GPU;
* the one exchange is the all-gather of per-chunk payload sizes (NCCL over
  NVLink/NVSwitch, or gloo on CPU), from which every rank knows the whole
  container layout (an exclusive scan);
* every rank then writes its span — its 25-byte records interleaved with its
  payloads, assembled on its device (``ebcc_fetch_container`` with
  ``EBCC_CONTAINER_BODY``) — straight into ONE shared host segment at its
  offset; rank 0 adds the 42-byte file header.  No payload byte is pickled or
  relayed through another rank.

``decompress`` mirrors it: rank 0 places the container in a shared segment,
every rank indexes it (native record walk), decodes its block of chunks on
its GPU and writes the float32 result into a shared output segment, which
rank 0 returns as the 4D array.

Errors are raised on every rank, the same exception everywhere: the one the
single-process API would raise (the first failing chunk / first non-finite
value in C order).  Custom ``chunk_shape`` grids are compressed by rank 0
alone through the single-process path (their chunks are not slices).
"""

from __future__ import annotations

import ctypes
import mmap
import os
import uuid

import numpy as np

from . import _lib
from .chunk import EbccParams
from .container import RECORD_DTYPE, pack_header, parse
from .core import _first_nonfinite, grid_from_array, pad_dims, tile_origins
from .errors import ArgumentError, EbccError, IngestError, ResidualInsufficient
from .pipeline import _check_streams, compress_batch, decompress_batch, default_levels
from .sharding import exchange_sizes, shard_bounds

__all__ = ["compress", "compress_shard", "decompress"]


def _dist():
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        raise ArgumentError("torch.distributed is not initialised (run under torchrun)")
    return dist


class _Segment:
    """A host buffer shared by the ranks of ``group`` (one node): a file in
    /dev/shm created by rank 0, mapped by every rank, unlinked once all have
    mapped it (the mappings stay valid)."""

    def __init__(self, nbytes: int, group=None):
        dist = _dist()
        self.rank = dist.get_rank(group)
        self.nbytes = max(1, int(nbytes))
        src = dist.get_global_rank(group, 0) if group is not None else 0
        path = None
        if self.rank == 0:
            path = os.path.join("/dev/shm", f"ebcc-{os.getpid()}-{uuid.uuid4().hex}")
            fd = os.open(path, os.O_CREAT | os.O_EXCL | os.O_RDWR, 0o600)
            os.ftruncate(fd, self.nbytes)
        obj = [path]
        dist.broadcast_object_list(obj, src=src, group=group)
        if self.rank != 0:
            fd = os.open(obj[0], os.O_RDWR)
        try:
            self.mm = mmap.mmap(fd, self.nbytes)
        finally:
            os.close(fd)
        dist.barrier(group)
        if self.rank == 0:
            os.unlink(path)
        self.view = np.frombuffer(self.mm, dtype=np.uint8)

    @property
    def ptr(self) -> int:
        return self.view.ctypes.data

    def close(self):
        self.view = None
        self.mm.close()


def _raise_first(errors):
    """Raise, on every rank, the first rank's error (rank order = chunk order)."""
    for e in errors:
        if e is not None:
            raise e


def _gather_errors(err, group):
    dist = _dist()
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, err, group=group)
    return out


def compress_shard(local_stack, dims, rel_error: float = 0.01, q: float = 1.0 - 1e-5,
                   group=None, ctx=None, coder=None, base_codec: str = "spiht") -> bytes | None:
    """Compress this rank's block of the default chunks of a ``dims`` grid.

    ``local_stack`` holds chunks ``shard_bounds(T*P, world, rank)`` (each an
    (H, W) slice, in tile order).  Every rank calls this collectively; rank
    0 returns the container bytes (byte-identical to
    ``paper_2510_22265_b200.compress`` of the whole array), the other ranks
    None.  ``coder(stack) -> (records[RECORD_DTYPE], payload uint8,
    offsets)`` replaces the device coder (the CPU multi-process tests use the
    oracle); its span is then assembled on the host.
    """
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dims = pad_dims(dims)
    t, p, h, w = dims
    n = t * p
    lo, hi = shard_bounds(n, world, rank)
    local = np.ascontiguousarray(local_stack, dtype=np.float32).reshape(-1, h, w)
    if local.shape[0] != hi - lo:
        raise ArgumentError(f"rank {rank} holds {local.shape[0]} chunks, its block is "
                            f"[{lo}, {hi})")
    params = EbccParams(epsilon_rel=float(rel_error), q=float(q))
    ctx = ctx or (_lib.context() if coder is None else None)
    err = None
    recs = None
    total = 0
    try:
        try:
            params.validate()
        except ArgumentError:
            bad = _first_nonfinite(local)  # ingest errors precede parameter errors
            if bad is not None:
                raise IngestError("non-finite", index=int(np.ravel_multi_index(bad, local.shape)))
            raise
        if hi > lo and coder is not None:
            recs, hpay, hoffs = coder(local)
            st = _lib.OK
        elif hi > lo:
            recs, _, total, st = compress_batch(local, params, ctx, fetch=False,
                                                base_codec=base_codec)
            if st == _lib.E_RESIDUAL:
                i = lo + int(np.flatnonzero(recs["status"] == _lib.E_RESIDUAL)[0])
                raise ResidualInsufficient(f"chunk at origin {(i // p, i % p, 0, 0)}: no "
                                           f"encoding reaches epsilon_rel={params.epsilon_rel} "
                                           "for this chunk")
    except IngestError as exc:
        flat = lo * h * w + int(exc.index)
        at = tuple(int(i) for i in np.unravel_index(flat, dims))
        err = IngestError(f"non-finite value at index {at}", index=at)
    except EbccError as exc:
        err = exc
    _raise_first(_gather_errors(err, group))

    local_sizes = (recs["base_len"] + recs["resid_len"]).astype(np.int64) if hi > lo \
        else np.zeros(0, np.int64)
    sizes = exchange_sizes(local_sizes, n, group)
    rec_span = 25 + sizes
    start = 42 + int(rec_span[:lo].sum())
    seg = _Segment(42 + int(rec_span.sum()), group)
    if hi > lo and coder is not None:
        pos = start
        for k in range(hi - lo):
            seg.view[pos: pos + 25] = np.frombuffer(recs[k: k + 1].tobytes(), np.uint8)
            ln = int(local_sizes[k])
            o = int(hoffs[k])
            seg.view[pos + 25: pos + 25 + ln] = hpay[o: o + ln]
            pos += 25 + ln
    elif hi > lo:
        r25 = np.zeros(hi - lo, RECORD_DTYPE)
        r25["mode"] = recs["mode"]
        r25["eps"] = params.epsilon_rel
        r25["q"] = params.q
        r25["vmin"] = recs["vmin"]
        r25["vmax"] = recs["vmax"]
        r25["base_len"] = recs["base_len"]
        r25["resid_len"] = recs["resid_len"]
        ctx.fetch_container_into(None, r25, total, seg.ptr + start,
                                 int(rec_span[lo:hi].sum()), _lib.CONTAINER_BODY)
    if rank == 0:
        from .container import VERSION, VERSION_EBCOT
        version = VERSION_EBCOT if base_codec == "ebcot" else VERSION
        seg.view[:42] = np.frombuffer(pack_header(dims, (1, 1, h, w), n, version), np.uint8)
    dist.barrier(group)
    out = seg.mm[:] if rank == 0 else None
    seg.close()
    return out


def compress(array, rel_error: float = 0.01, q: float = 1.0 - 1e-5, chunk_shape=None,
             group=None, base_codec: str = "spiht") -> bytes | None:
    """``paper_2510_22265_b200.compress`` over the ranks of ``group``: every
    rank passes the same (T, P, H, W) array (or a view of it; a rank reads
    only its block); rank 0 returns the container, the others None.
    ``base_codec="ebcot"``: the opt-in JPEG2000-style base layer (version 2)."""
    dist = _dist()
    data = np.asarray(array)
    dims = pad_dims(data.shape)
    if chunk_shape is not None and tuple(pad_dims(chunk_shape)) != (1, 1) + dims[2:]:
        from .api import compress as single
        out = single(array, rel_error, q, chunk_shape, base_codec) \
            if dist.get_rank(group) == 0 else None
        dist.barrier(group)
        return out
    if data.size == 0:
        grid_from_array(data)  # the reference's IngestError("empty input array")
    t, p, h, w = dims
    lo, hi = shard_bounds(t * p, dist.get_world_size(group), dist.get_rank(group))
    return compress_shard(data.reshape(t * p, h, w)[lo:hi], dims, rel_error, q, group,
                          base_codec=base_codec)


def decompress(buf, group=None) -> np.ndarray | None:
    """``paper_2510_22265_b200.decompress`` over the ranks of ``group``:
    ``buf`` (container bytes) is read on rank 0 only; every rank decodes its
    block of chunks on its GPU; rank 0 returns the 4D float32 array (backed
    by a shared segment), the other ranks None."""
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ln = [len(buf) if rank == 0 else 0]
    dist.broadcast_object_list(ln, src=dist.get_global_rank(group, 0) if group is not None
                               else 0, group=group)
    seg = _Segment(ln[0], group)
    if rank == 0 and ln[0]:
        ctypes.memmove(seg.ptr, bytes(buf) if not isinstance(buf, bytes) else buf, ln[0])
    dist.barrier(group)
    err = None
    parsed = None
    try:
        parsed = parse(seg.mm)
    except EbccError as exc:
        err = exc
    _raise_first(_gather_errors(err, group))
    dims, chunk_shape, recs, offs, data = parsed
    t, p, h, w = (int(d) for d in dims)
    if tuple(int(c) for c in chunk_shape[:2]) != (1, 1) or chunk_shape[2] < h \
            or chunk_shape[3] < w:
        out = None
        if rank == 0:
            from .pipeline import records_to_grid
            out = records_to_grid(dims, chunk_shape, recs, offs, bytes(seg.mm[:]))
        dist.barrier(group)
        seg.close()
        return out
    n = t * p
    lo, hi = shard_bounds(n, world, rank)
    oseg = _Segment(4 * n * h * w, group)
    err = None
    try:
        if hi > lo:
            local = np.frombuffer(oseg.mm, dtype=np.float32, count=(hi - lo) * h * w,
                                  offset=4 * lo * h * w).reshape(hi - lo, h, w)
            lrecs, loffs = recs[lo:hi], offs[lo:hi]
            levels = _check_streams(seg.view, lrecs, loffs, h, w)
            groups = {}
            if levels >= 0:
                groups[levels or default_levels(h, w)] = np.arange(hi - lo)
            else:
                for k in range(hi - lo):
                    lv = _check_streams(seg.view, lrecs[k:k + 1], loffs[k:k + 1], h, w)
                    groups.setdefault(lv or default_levels(h, w), []).append(k)
            for lv, idx in groups.items():
                idx = np.asarray(idx)
                r = np.zeros(len(idx), dtype=_lib.REC_DTYPE)
                for f in ("mode", "base_len", "resid_len"):
                    r[f] = lrecs[f][idx]
                r["vmin"] = lrecs["vmin"][idx].astype(np.float64)
                r["vmax"] = lrecs["vmax"][idx].astype(np.float64)
                if len(idx) == hi - lo:
                    decompress_batch(seg.view, loffs, r, h, w, lv, out=local)
                else:
                    local[idx] = decompress_batch(seg.view, loffs[idx], r, h, w, lv)
    except EbccError as exc:
        err = exc
    local = None  # drop the views of the shared segments before unmapping
    _raise_first(_gather_errors(err, group))
    dist.barrier(group)
    seg.close()
    if rank != 0:
        oseg.close()
        return None
    out = np.frombuffer(oseg.mm, dtype=np.float32, count=n * h * w).reshape(t, p, h, w)
    return out


def decompress_shard(buf, group=None):
    """Alias of :func:`decompress` (rank 0 passes the container)."""
    return decompress(buf, group)
