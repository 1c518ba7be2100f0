"""The EBCC container: byte-identical to the reference's file format.

Layout (little endian; pkg/src/ebcc/container.py:1-27):

    file header (42 B)  '<4sH4I4II'  magic 'EBCC', version 1, dims[4],
                                     chunk_shape[4], chunk_count
    per chunk (25 B)    '<BffffII'   mode, epsilon_rel, q, vmin, vmax,
                                     base_len, residual_len
                        then base_len + residual_len payload bytes

Chunks follow row-major tile order, so dims + chunk_shape fix every chunk's
origin and block shape.  Parsing raises FormatError(offset) on structural
damage and UnsupportedVersion on a version mismatch, at the same offsets as
the reference (container.py:82-145).  Records are packed with a numpy
structured dtype so large grids serialise without a Python loop per field.
"""

from __future__ import annotations

import io
import struct

import numpy as np

from .chunk import CompressedChunk, Mode
from .core import block_count, block_shape_at, pad_dims, tile_origins
from .errors import FormatError, IoError, UnsupportedVersion

MAGIC = b"EBCC"
VERSION = 1
# version 2: the same layout with JPEG2000-style ('J2') base streams (the
# opt-in base_codec="ebcot"; the reference reads only version 1)
VERSION_EBCOT = 2
VERSIONS = (VERSION, VERSION_EBCOT)

HEADER = struct.Struct("<4sH4I4II")
RECORD = struct.Struct("<BffffII")
RECORD_DTYPE = np.dtype([("mode", "u1"), ("eps", "<f4"), ("q", "<f4"), ("vmin", "<f4"),
                         ("vmax", "<f4"), ("base_len", "<u4"), ("resid_len", "<u4")])
assert RECORD_DTYPE.itemsize == RECORD.size == 25


def pack_header(dims, chunk_shape, count: int, version: int = VERSION) -> bytes:
    return HEADER.pack(MAGIC, version, *dims, *chunk_shape, count)


def pack_record(mode, eps, q, vmin, vmax, base_len, resid_len) -> bytes:
    return RECORD.pack(int(mode), eps, q, vmin, vmax, int(base_len), int(resid_len))


def assemble(dims, chunk_shape, records: np.ndarray, payload: np.ndarray,
             offsets: np.ndarray, version: int = VERSION) -> bytes:
    """Container bytes from a record array and one contiguous payload buffer.

    ``records`` has RECORD_DTYPE; chunk i's payload is
    payload[offsets[i] : offsets[i] + base_len + resid_len].
    """
    dims = pad_dims(dims)
    chunk_shape = pad_dims(chunk_shape)
    expected = block_count(dims, chunk_shape)
    if len(records) != expected:
        raise FormatError(f"grid {dims} with chunk shape {chunk_shape} needs {expected} "
                          f"chunks, got {len(records)}")
    parts = [pack_header(dims, chunk_shape, len(records), version)]
    rec_bytes = records.astype(RECORD_DTYPE, copy=False).tobytes()
    lens = records["base_len"].astype(np.int64) + records["resid_len"].astype(np.int64)
    for i in range(len(records)):
        parts.append(rec_bytes[25 * i: 25 * i + 25])
        o = int(offsets[i])
        parts.append(payload[o: o + int(lens[i])].tobytes())
    return b"".join(parts)


def write_file(chunks, dims, chunk_shape, sink, version: int = VERSION) -> int:
    dims = pad_dims(dims)
    chunk_shape = pad_dims(chunk_shape)
    expected = block_count(dims, chunk_shape)
    if len(chunks) != expected:
        raise FormatError(f"grid {dims} with chunk shape {chunk_shape} needs {expected} "
                          f"chunks, got {len(chunks)}")
    out = io.BytesIO()
    out.write(pack_header(dims, chunk_shape, len(chunks), version))
    for cc in chunks:
        out.write(pack_record(cc.mode, cc.epsilon_rel, cc.q, cc.vmin, cc.vmax, cc.base_len,
                              cc.residual_len))
        out.write(cc.payload)
    blob = out.getvalue()
    try:
        if hasattr(sink, "write"):
            sink.write(blob)
        else:
            with open(sink, "wb") as fh:
                fh.write(blob)
    except OSError as exc:
        raise IoError(f"cannot write output: {exc}") from exc
    return len(blob)


def write_bytes(chunks, dims, chunk_shape, version: int = VERSION) -> bytes:
    sink = io.BytesIO()
    write_file(chunks, dims, chunk_shape, sink, version)
    return sink.getvalue()


def _load(source) -> bytes:
    import mmap
    if isinstance(source, mmap.mmap):
        return source  # a shared segment (distributed.decompress): indexed in place
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source)
    if hasattr(source, "read"):
        return source.read()
    try:
        with open(source, "rb") as fh:
            return fh.read()
    except OSError as exc:
        raise IoError(f"cannot read input: {exc}") from exc


def parse(source):
    """Validate a container and index it without copying payloads.

    Returns (dims, chunk_shape, records, payload_offsets, data) where
    records is a RECORD_DTYPE array and payload_offsets[i] is the absolute
    offset of chunk i's payload inside ``data``.
    """
    data = _load(source)
    if len(data) < HEADER.size:
        raise FormatError("file shorter than header", offset=len(data))
    head = HEADER.unpack_from(data, 0)
    if head[0] != MAGIC:
        raise FormatError(f"bad magic {head[0]!r}", offset=0)
    if head[1] not in VERSIONS:
        raise UnsupportedVersion(f"unsupported format version {head[1]}", offset=4)
    dims = tuple(head[2:6])
    chunk_shape = tuple(head[6:10])
    count = head[10]
    if min(chunk_shape) < 1:
        raise FormatError(f"bad chunk shape {chunk_shape}", offset=22)
    expected = block_count(dims, chunk_shape)
    if count != expected:
        raise FormatError(f"chunk count {count} inconsistent with tiling ({expected})",
                          offset=42)
    recs, offs = index_records(data, count)
    return dims, chunk_shape, recs, offs, data


_PARSE_ERRORS = {1: "truncated chunk record", 3: "truncated chunk payload"}


def index_records(data, count: int):
    """The record walk of read_file (container.py:82-145) in the native
    library (``ebcc_parse_records``): RECORD_DTYPE records and the absolute
    payload offset of each chunk; FormatError at the reference's offsets."""
    import ctypes

    from . import _lib
    lib = _lib.load()
    recs = np.empty(count, dtype=RECORD_DTYPE)
    offs = np.empty(count, dtype=np.int64)
    view = np.frombuffer(data, dtype=np.uint8)
    eoff = ctypes.c_int64(-1)
    aux = ctypes.c_int32(0)
    st = lib.ebcc_parse_records(view.ctypes.data if view.size else None, view.size, count,
                                recs.ctypes.data if count else None,
                                offs.ctypes.data if count else None, ctypes.byref(eoff),
                                ctypes.byref(aux))
    if st == _lib.OK:
        return recs, offs
    pos = int(eoff.value)
    if st == _lib.E_FORMAT:
        if aux.value == 2:
            raise FormatError(f"unknown chunk mode {int(view[pos])}", offset=pos)
        if aux.value == 4:
            raise FormatError(f"{view.size - pos} trailing bytes after last chunk", offset=pos)
        raise FormatError(_PARSE_ERRORS[aux.value], offset=pos)
    raise FormatError("cannot index container records", offset=HEADER.size)


def read_file(source):
    """Parse into CompressedChunk objects (reference container.read_file)."""
    dims, chunk_shape, recs, offs, data = parse(source)
    chunks = []
    for i, origin in enumerate(tile_origins(dims, chunk_shape)):
        rec = recs[i]
        t, p, h, w = block_shape_at(origin, dims, chunk_shape)
        n = int(rec["base_len"]) + int(rec["resid_len"])
        chunks.append(CompressedChunk(
            mode=Mode(int(rec["mode"])), epsilon_rel=float(rec["eps"]), q=float(rec["q"]),
            vmin=float(rec["vmin"]), vmax=float(rec["vmax"]), base_len=int(rec["base_len"]),
            residual_len=int(rec["resid_len"]), payload=data[offs[i]: offs[i] + n],
            rows=t * p * h, cols=w, block_shape=(t, p, h, w), origin=origin))
    return chunks, dims, chunk_shape
