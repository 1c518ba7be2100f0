"""Chunk pipeline: the reference's compress/decompress entry points, served by
the B200 library.

Drop-in for pkg/src/ebcc/pipeline.py: ``compress_grid`` (pipeline.py:358-367)
and ``decompress_grid`` (370-379) keep their signatures, chunk order, error
types and "chunk at origin ..." messages, but instead of a serial Python loop
over ``compress_chunk`` they hand every same-shape group of chunks to ONE
``ebcc_compress`` / ``ebcc_decompress`` call (include/ebcc_gpu.h), which runs
the whole per-chunk algorithm — normalise, DWT, SPIHT, the three feedback
searches, candidate choice — on the device.  ``compress_chunk`` /
``decompress_chunk`` are the one-chunk special cases.

Nothing here computes on the CPU: without the CUDA library every call raises
``DeviceError``.
"""

from __future__ import annotations

import struct

import numpy as np

from . import _lib
from .chunk import CompressedChunk, EbccParams, Mode
from .container import RECORD_DTYPE
from .core import (Chunk, GridArray, block_shape_at, flatten_chunk, iter_blocks, tile_origins,
                   unflatten_chunk)
from .errors import ArgumentError, EbccError, FormatError, IngestError, ResidualInsufficient

__all__ = ["Mode", "EbccParams", "CompressedChunk", "compress_chunk", "decompress_chunk",
           "compress_grid", "decompress_grid", "compress_batch", "decompress_batch",
           "default_levels"]

HEADER_SIZE = 12
_SP_HEADER = struct.Struct("<2sbBII")


def default_levels(rows: int, cols: int) -> int:
    """dwt.default_levels (dwt.py:35-41)."""
    m = min(rows, cols)
    if m < 2:
        return 1
    return max(1, min(5, int(m).bit_length() - 1 - 2))


# ---------------------------------------------------------------------------
# batched device calls

def compress_batch(stack: np.ndarray, params: EbccParams, ctx=None, fetch: bool = True,
                   full_search: bool = False, base_codec: str = "spiht"):
    """Compress a (n, rows, cols) float32 stack of chunks on the device.

    Returns (records[REC_DTYPE], offsets int64[n], payload uint8[total],
    status).  Raises ArgumentError for bad params; per-chunk
    ResidualInsufficient is reported through records['status'] and status.
    With ``fetch=False`` the payload stays on the device (payload is the int
    total) for :meth:`_lib.Context.fetch_container`.  ``full_search`` runs
    every probe of the reference's searches (the default stops a search whose
    candidate can no longer be chosen: same bytes, fewer probes).
    ``base_codec="ebcot"`` selects the opt-in JPEG2000-style base layer
    ('J2' streams, container version 2; the reference has no such layer).
    """
    if base_codec not in _lib.BASE_CODECS:
        raise ArgumentError(f"unknown base codec {base_codec!r}")
    ctx = ctx or _lib.context()
    stack = np.ascontiguousarray(stack, dtype=np.float32)
    n, rows, cols = stack.shape
    recs, offs, total, st = ctx.compress(stack, n, rows, cols, params.epsilon_rel, params.q,
                                         params.r0, params.search_tol,
                                         flags=(_lib.FULL_SEARCH if full_search else 0) |
                                         _lib.BASE_CODECS[base_codec])
    if st not in (_lib.OK, _lib.E_RESIDUAL):
        ctx.raise_for(st, "ebcc_compress")
    if not fetch:
        return recs, offs, total, st
    payload = np.empty(max(total, 1), dtype=np.uint8)
    if st == _lib.OK and total:
        ctx.fetch_payload(payload)
    return recs, offs, payload[:total], st


def decompress_batch(payload: np.ndarray, offsets: np.ndarray, recs: np.ndarray, rows: int,
                     cols: int, levels: int, out: np.ndarray | None = None, ctx=None):
    """Decompress same-shape chunks into a (n, rows, cols) float32 array."""
    ctx = ctx or _lib.context()
    n = len(recs)
    if out is None:
        out = np.empty((n, rows, cols), dtype=np.float32)
    if n == 0:
        return out
    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    if payload.size == 0:
        payload = np.zeros(1, np.uint8)
    ctx.decompress(payload, np.ascontiguousarray(offsets, np.int64),
                   np.ascontiguousarray(recs), rows, cols, levels, out)
    return out


# ---------------------------------------------------------------------------
# reference-shaped API

def _chunk_error(origin, exc: EbccError):
    exc.args = (f"chunk at origin {origin}: {exc.args[0] if exc.args else exc}",)
    return exc


def _compressed_from_records(chunks, recs, offs, payload, params):
    out = []
    for ch, rec, off in zip(chunks, recs, offs):
        n = int(rec["base_len"]) + int(rec["resid_len"])
        out.append(CompressedChunk(
            mode=Mode(int(rec["mode"])), epsilon_rel=params.epsilon_rel, q=params.q,
            vmin=float(rec["vmin"]), vmax=float(rec["vmax"]), base_len=int(rec["base_len"]),
            residual_len=int(rec["resid_len"]), payload=payload[off: off + n].tobytes(),
            rows=ch.rows, cols=ch.cols, block_shape=ch.block_shape, origin=ch.origin))
    return out


def _each_group(fn, groups: dict, ctx):
    """fn over the same-shape chunk groups, in group order.  (Running the
    groups concurrently, one worker thread and library context each, measured
    slower once each context keeps a workspace per chunk shape: 199 vs 152 ms
    for 37 levels in 256x512 chunks; the groups contend for the SMs.)"""
    return [fn(it) for it in groups.items()]


def compress_chunks(chunks: list, params: EbccParams, ctx=None,
                    base_codec: str = "spiht") -> list:
    """Compress a list of flattened Chunk objects (any shapes), tile order kept."""
    if not chunks:
        return []
    try:
        params.validate()
    except ArgumentError as exc:
        raise _chunk_error(chunks[0].origin, exc)
    for ch in chunks:
        if ch.normalized:
            raise _chunk_error(ch.origin, ArgumentError("compress_chunk expects an unnormalized chunk"))
    groups: dict = {}
    for i, ch in enumerate(chunks):
        groups.setdefault((ch.rows, ch.cols), []).append(i)
    result = [None] * len(chunks)
    failed = []

    def run(item):
        (rows, cols), idx = item
        stack = np.empty((len(idx), rows, cols), dtype=np.float32)
        for k, i in enumerate(idx):
            stack[k] = chunks[i].values
        return compress_batch(stack, params, ctx, base_codec=base_codec)

    for ((rows, cols), idx), (recs, offs, payload, st) in zip(groups.items(),
                                                              _each_group(run, groups, ctx)):
        if st == _lib.E_RESIDUAL:
            failed.extend(i for k, i in enumerate(idx) if recs[k]["status"] == _lib.E_RESIDUAL)
            continue
        for k, cc in enumerate(_compressed_from_records([chunks[i] for i in idx], recs, offs,
                                                        payload, params)):
            result[idx[k]] = cc
    if failed:
        first = min(failed)
        raise _chunk_error(chunks[first].origin, ResidualInsufficient(
            f"no encoding reaches epsilon_rel={params.epsilon_rel} for this chunk"))
    return result


def compress_chunk(chunk: Chunk, params: EbccParams, ctx=None) -> CompressedChunk:
    """pipeline.compress_chunk (pipeline.py:277-329) — one-chunk batch."""
    try:
        return compress_chunks([chunk], params, ctx)[0]
    except EbccError as exc:
        # the reference raises without the origin prefix for a bare chunk
        msg = str(exc)
        prefix = f"chunk at origin {chunk.origin}: "
        if msg.startswith(prefix):
            exc.args = (msg[len(prefix):],)
        raise


def compress_grid(grid: GridArray, params: EbccParams, ctx=None,
                  base_codec: str = "spiht") -> list:
    """pipeline.compress_grid (pipeline.py:358-367), batched on the device."""
    chunks = [flatten_chunk(block, origin) for origin, block in iter_blocks(grid)]
    return compress_chunks(chunks, params, ctx, base_codec)


def _parse_sp(data: bytes, rows: int, cols: int, what: str):
    if len(data) < HEADER_SIZE:
        raise FormatError(f"stream shorter than {HEADER_SIZE}-byte header", offset=len(data))
    magic, n_max, levels, r, c = _SP_HEADER.unpack_from(data, 0)
    # (a base stream may be 'J2': the opt-in JPEG2000-style layer, container v2)
    if magic != b"SP" and not (what == "base" and magic == b"J2"):
        raise FormatError(f"bad stream magic {magic!r}", offset=0)
    if r < 1 or c < 1 or levels < 1:
        raise FormatError(f"bad stream dimensions {r}x{c}/{levels}", offset=2)
    if (r, c) != (rows, cols):
        raise FormatError(f"{what} stream shape {(r, c)} does not match chunk {(rows, cols)}")
    return n_max, levels


def _validate_chunk(cc: CompressedChunk) -> int:
    """decompress_chunk's structural checks (pipeline.py:336-353); returns levels."""
    if cc.mode == Mode.CONSTANT:
        return 0
    if cc.base_len + cc.residual_len != len(cc.payload):
        raise FormatError(f"payload length {len(cc.payload)} does not match base_len + "
                          f"residual_len = {cc.base_len + cc.residual_len}",
                          offset=len(cc.payload))
    _, levels = _parse_sp(cc.payload[: cc.base_len], cc.rows, cc.cols, "base")
    if cc.mode == Mode.TWO_LAYER and cc.residual_len > 0:
        _, rl = _parse_sp(cc.payload[cc.base_len:], cc.rows, cc.cols, "residual")
        if rl != levels:
            raise FormatError("residual stream levels differ from the base stream's", offset=3)
    if levels > 5:
        raise FormatError(f"unsupported decomposition depth {levels}", offset=3)
    return levels


def decompress_chunks(chunks: list, ctx=None) -> list:
    """Decompress CompressedChunk objects; returns a list of (rows, cols) f32."""
    levels = [_validate_chunk(cc) for cc in chunks]
    groups: dict = {}
    for i, cc in enumerate(chunks):
        lv = levels[i] if levels[i] else default_levels(cc.rows, cc.cols)
        groups.setdefault((cc.rows, cc.cols, lv), []).append(i)
    out = [None] * len(chunks)

    def run(item):
        (rows, cols, lv), idx = item
        recs = np.zeros(len(idx), dtype=_lib.REC_DTYPE)
        offs = np.zeros(len(idx), dtype=np.int64)
        parts = []
        pos = 0
        for k, i in enumerate(idx):
            cc = chunks[i]
            recs[k]["mode"] = int(cc.mode)
            recs[k]["vmin"] = cc.vmin
            recs[k]["vmax"] = cc.vmax
            recs[k]["base_len"] = cc.base_len
            recs[k]["resid_len"] = cc.residual_len
            offs[k] = pos
            parts.append(cc.payload)
            pos += len(cc.payload)
        payload = np.frombuffer(b"".join(parts), dtype=np.uint8) if pos else np.zeros(1, np.uint8)
        return decompress_batch(payload, offs, recs, rows, cols, lv, ctx=ctx)

    # serial: concurrent groups measured slower here (host-side staging and
    # per-chunk Python work dominate this path)
    for item in groups.items():
        res = run(item)
        for k, i in enumerate(item[1]):
            out[i] = res[k]
    return out


def decompress_chunk(cc: CompressedChunk, ctx=None) -> np.ndarray:
    """pipeline.decompress_chunk (pipeline.py:332-355)."""
    return decompress_chunks([cc], ctx)[0]


def decompress_grid(chunks, dims, chunk_shape=None, ctx=None) -> np.ndarray:
    """pipeline.decompress_grid (pipeline.py:370-379)."""
    data = np.empty(tuple(dims), dtype=np.float32)
    values = decompress_chunks(list(chunks), ctx)
    for cc, v in zip(chunks, values):
        block = unflatten_chunk(v, cc.block_shape)
        t0, p0, h0, w0 = cc.origin
        t, p, h, w = cc.block_shape
        data[t0: t0 + t, p0: p0 + p, h0: h0 + h, w0: w0 + w] = block
    return data


# ---------------------------------------------------------------------------
# container-level fast paths used by api.compress / api.decompress

def grid_to_records(grid: GridArray, params: EbccParams, ctx=None, orig_shape=None,
                    container: bool = False, base_codec: str = "spiht"):
    """Compress a grid straight to (records[RECORD_DTYPE], payload, offsets).

    Default chunking (one 2D slice per (t, p)) is fed to the device without a
    host-side gather, and the non-finite scan happens on the device (reported
    as IngestError with the index in ``orig_shape``, the caller's array
    shape).  Error semantics and their order equal the reference's
    (ingest before parameter validation, core.py:89-105 / pipeline.py:54).
    With ``container=True`` the result is the container bytes, assembled on
    the device for default chunking.
    """
    t, p, h, w = grid.dims
    shape = tuple(orig_shape) if orig_shape is not None else tuple(grid.dims)
    if tuple(grid.chunk_shape) == (1, 1, h, w):
        origins = tile_origins(grid.dims, grid.chunk_shape)
        try:
            params.validate()
        except ArgumentError as exc:
            from .core import _require_finite
            _require_finite(grid.data.reshape(shape))
            raise _chunk_error(origins[0], exc)
        stack = grid.data.reshape(t * p, h, w)
        ctx = ctx or _lib.context()
        try:
            recs, offs, payload, st = compress_batch(stack, params, ctx, fetch=not container,
                                                     base_codec=base_codec)
        except IngestError as exc:
            at = tuple(int(i) for i in np.unravel_index(int(exc.index), shape))
            raise IngestError(f"non-finite value at index {at}", index=at) from None
        if st == _lib.E_RESIDUAL:
            bad = int(np.flatnonzero(recs["status"] == _lib.E_RESIDUAL)[0])
            raise _chunk_error(origins[bad], ResidualInsufficient(
                f"no encoding reaches epsilon_rel={params.epsilon_rel} for this chunk"))
        out = np.zeros(len(recs), dtype=RECORD_DTYPE)
        out["mode"] = recs["mode"]
        out["eps"] = params.epsilon_rel
        out["q"] = params.q
        out["vmin"] = recs["vmin"]
        out["vmax"] = recs["vmax"]
        out["base_len"] = recs["base_len"]
        out["resid_len"] = recs["resid_len"]
        if container:
            from .container import VERSION, VERSION_EBCOT, pack_header
            version = VERSION_EBCOT if base_codec == "ebcot" else VERSION
            return ctx.fetch_container(pack_header(grid.dims, grid.chunk_shape, len(out), version),
                                       out, payload)
        return out, payload, offs, recs
    from .core import _require_finite
    _require_finite(grid.data.reshape(shape))
    chunks = compress_grid(grid, params, ctx, base_codec)
    out = np.zeros(len(chunks), dtype=RECORD_DTYPE)
    offs = np.zeros(len(chunks), dtype=np.int64)
    pos = 0
    for i, cc in enumerate(chunks):
        out[i] = (int(cc.mode), cc.epsilon_rel, cc.q, cc.vmin, cc.vmax, cc.base_len,
                  cc.residual_len)
        offs[i] = pos
        pos += len(cc.payload)
    payload = np.frombuffer(b"".join(cc.payload for cc in chunks), np.uint8) if pos else \
        np.zeros(0, np.uint8)
    if container:
        from .container import VERSION, VERSION_EBCOT, assemble
        return assemble(grid.dims, grid.chunk_shape, out, payload, offs,
                        VERSION_EBCOT if base_codec == "ebcot" else VERSION)
    return out, payload, offs, None


def records_to_grid(dims, chunk_shape, recs: np.ndarray, offs: np.ndarray, data: bytes,
                    ctx=None) -> np.ndarray:
    """Decompress a parsed container into the 4D float32 array."""
    dims = tuple(int(d) for d in dims)
    chunk_shape = tuple(int(c) for c in chunk_shape)
    t, p, h, w = dims
    if len(recs) == 0:
        return np.empty(dims, np.float32)
    if chunk_shape[0] == 1 and chunk_shape[1] == 1 and chunk_shape[2] >= h and chunk_shape[3] >= w:
        # one (h, w) chunk per (t, p): validate headers vectorised, decode in place
        buf = np.frombuffer(data, dtype=np.uint8)
        mode = recs["mode"].astype(np.int64)
        blen = recs["base_len"].astype(np.int64)
        rlen = recs["resid_len"].astype(np.int64)
        levels = _check_streams(buf, recs, offs, h, w)
        if levels < 0:  # chunks of different depths
            return _records_to_grid_slow(dims, chunk_shape, recs, offs, data, ctx)
        out = _lib.host_empty(dims, np.float32)
        lrec = np.zeros(len(recs), dtype=_lib.REC_DTYPE)
        lrec["mode"] = mode
        lrec["vmin"] = recs["vmin"].astype(np.float64)
        lrec["vmax"] = recs["vmax"].astype(np.float64)
        lrec["base_len"] = blen
        lrec["resid_len"] = rlen
        decompress_batch(buf, offs, lrec, h, w, levels or default_levels(h, w),
                         out=out.reshape(t * p, h, w), ctx=ctx)
        return out
    return _records_to_grid_slow(dims, chunk_shape, recs, offs, data, ctx)


def _check_streams(buf: np.ndarray, recs: np.ndarray, offs: np.ndarray, rows: int,
                   cols: int) -> int:
    """Stream-header checks of every same-shape chunk in the native library
    (``ebcc_check_streams``); returns the common level count (0: all
    constant), -1 for mixed depths, and raises the reference's FormatError
    for the first bad chunk."""
    import ctypes
    lib = _lib.load()
    recs = np.ascontiguousarray(recs)
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    lv = ctypes.c_int32(0)
    bad = ctypes.c_int64(-1)
    n = len(recs)
    st = lib.ebcc_check_streams(buf.ctypes.data if buf.size else None, buf.size,
                                recs.ctypes.data if n else None, offs.ctypes.data if n else None,
                                n, rows, cols, ctypes.byref(lv), ctypes.byref(bad))
    if st == _lib.OK:
        return int(lv.value)
    if st == _lib.E_ARGUMENT and bad.value >= 0:
        return -1
    i = int(bad.value)
    # the exact reference message for that chunk
    _validate_payload(buf, int(offs[i]), int(recs["base_len"][i]), int(recs["resid_len"][i]),
                      int(recs["mode"][i]), rows, cols)
    raise FormatError("bad stream header", offset=int(offs[i]))


def _validate_payload(data, off, blen, rlen, mode, rows, cols) -> int:
    mv = memoryview(data)  # header checks without copying the streams
    _, levels = _parse_sp(mv[off: off + blen], rows, cols, "base")
    if mode == int(Mode.TWO_LAYER) and rlen > 0:
        _, rl = _parse_sp(mv[off + blen: off + blen + rlen], rows, cols, "residual")
        if rl != levels:
            raise FormatError("residual stream levels differ from the base stream's", offset=3)
    if levels > 5:
        raise FormatError(f"unsupported decomposition depth {levels}", offset=3)
    return levels


def _records_to_grid_slow(dims, chunk_shape, recs, offs, data, ctx):
    """Any chunking: chunks grouped by (rows, cols, levels), each group decoded
    by one device call straight from the container bytes (records' offsets
    index ``data``; no per-chunk payload copies), blocks scattered back in
    tile order."""
    origins = tile_origins(dims, chunk_shape)
    buf = np.frombuffer(data, dtype=np.uint8)
    mode = recs["mode"].astype(np.int64)
    blen = recs["base_len"].astype(np.int64)
    rlen = recs["resid_len"].astype(np.int64)
    shapes = [block_shape_at(o, dims, chunk_shape) for o in origins]
    groups: dict = {}
    for i, (tt, pp, hh, ww) in enumerate(shapes):
        rows, cols = tt * pp * hh, ww
        lv = 0
        if mode[i] != int(Mode.CONSTANT):
            lv = _validate_payload(data, int(offs[i]), int(blen[i]), int(rlen[i]), int(mode[i]),
                                   rows, cols)
        groups.setdefault((rows, cols, lv or default_levels(rows, cols)), []).append(i)
    out = np.empty(tuple(dims), dtype=np.float32)
    for (rows, cols, lv), idx in groups.items():
        idx = np.asarray(idx)
        lrec = np.zeros(len(idx), dtype=_lib.REC_DTYPE)
        lrec["mode"] = mode[idx]
        lrec["vmin"] = recs["vmin"][idx].astype(np.float64)
        lrec["vmax"] = recs["vmax"][idx].astype(np.float64)
        lrec["base_len"] = blen[idx]
        lrec["resid_len"] = rlen[idx]
        res = decompress_batch(buf, np.ascontiguousarray(offs[idx], dtype=np.int64), lrec, rows,
                               cols, lv, ctx=ctx)
        for k, i in enumerate(idx):
            t0, p0, h0, w0 = origins[i]
            t, p, h, w = shapes[i]
            out[t0: t0 + t, p0: p0 + p, h0: h0 + h, w0: w0 + w] = res[k].reshape(t, p, h, w)
    return out
