"""CPU tests of the host side: the C ABI surface, the container format, the
grid model, and the sharded (multi-process, gloo) container assembly."""

import ctypes
import io
import os
import re

import numpy as np
import pytest

import golden_inputs as gi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------------------
# C ABI
def _header_functions():
    txt = open(os.path.join(REPO, "include", "ebcc_gpu.h")).read()
    return sorted(set(re.findall(r"\b(ebcc_[a-z_]+)\s*\(", txt)))


def test_abi_library_exports_every_declared_symbol():
    from paper_2510_22265_b200 import _lib
    path = _lib.LIB_PATH
    assert os.path.exists(path), "build() must produce the in-tree libebcc_gpu.so"
    lib = ctypes.CDLL(path)
    declared = _header_functions()
    assert declared, "no ebcc_* functions found in include/ebcc_gpu.h"
    for name in declared:
        assert hasattr(lib, name), f"{name} declared but not exported"
    assert sorted(_lib.EXPORTS) == declared


def test_abi_version_and_fail_loudly_without_gpu():
    from paper_2510_22265_b200 import _lib
    lib = _lib.load()
    assert lib.ebcc_abi_version() == 1
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2510_22265_b200 as ebcc
    with pytest.raises(ebcc.DeviceError):
        ebcc.compress(np.ones((8, 8), np.float32))


def test_abi_rejects_bad_params_before_touching_the_device():
    """EbccParams validation (pipeline.py:54-62) happens host side."""
    import paper_2510_22265_b200 as ebcc
    for kw in (dict(rel_error=0.0), dict(rel_error=1.0), dict(q=0.0), dict(q=1.5)):
        with pytest.raises(ebcc.ArgumentError, match="origin"):
            ebcc.compress(np.ones((8, 8), np.float32) * np.arange(8, dtype=np.float32), **kw)


# ---------------------------------------------------------------------------
# container (byte-identical to the reference format)
def test_golden_containers_reparse_bitwise(golden_chunks):
    from paper_2510_22265_b200.container import read_file, write_bytes, parse, assemble
    for case in golden_chunks["chunks"] + golden_chunks["grids"]:
        if not case.get("container"):
            continue
        blob = bytes.fromhex(case["container"])
        chunks, dims, cs = read_file(blob)
        assert write_bytes(chunks, dims, cs) == blob
        d2, cs2, recs, offs, data = parse(blob)
        assert assemble(d2, cs2, recs, np.frombuffer(data, np.uint8), offs) == blob
        assert [int(c.mode) for c in chunks] == case["modes"]


def test_container_fault_injection(golden_chunks):
    from paper_2510_22265_b200.container import read_file
    from paper_2510_22265_b200.errors import FormatError, UnsupportedVersion
    blobs = [bytes.fromhex(c["container"]) for c in golden_chunks["grids"]]
    rng = np.random.default_rng(13)
    for blob in blobs:
        for cut in range(0, len(blob), max(1, len(blob) // 40)):
            with pytest.raises((FormatError, UnsupportedVersion)):
                read_file(blob[:cut])
        for _ in range(25):
            bad = bytearray(blob)
            bad[int(rng.integers(0, len(blob)))] ^= 0xFF
            try:
                read_file(bytes(bad))
            except (FormatError, UnsupportedVersion):
                pass


def test_container_errors_and_io(tmp_path):
    from paper_2510_22265_b200.container import read_file, write_bytes, write_file
    from paper_2510_22265_b200.errors import FormatError, IoError, UnsupportedVersion
    blob = write_bytes([], (0, 0, 0, 0), (1, 1, 1, 1))
    assert len(blob) == 42
    chunks, dims, _ = read_file(blob)
    assert chunks == [] and dims == (0, 0, 0, 0)
    with pytest.raises(FormatError):
        read_file(b"XBCC" + blob[4:])
    with pytest.raises(UnsupportedVersion):
        read_file(blob[:4] + b"\x03\x00" + blob[6:])
    # version 2 = this repository's opt-in JPEG2000-style base layer
    assert read_file(blob[:4] + b"\x02\x00" + blob[6:])[1] == (0, 0, 0, 0)
    with pytest.raises(IoError):
        read_file("/nonexistent/x.ebcc")
    p = tmp_path / "e.ebcc"
    assert write_file([], (0, 0, 0, 0), (1, 1, 1, 1), str(p)) == 42
    buf = io.BytesIO()
    write_file([], (0, 0, 0, 0), (1, 1, 1, 1), buf)
    assert buf.getvalue() == p.read_bytes()


# ---------------------------------------------------------------------------
# grid model (core.py)
def test_ingest_validation():
    from paper_2510_22265_b200 import core
    from paper_2510_22265_b200.errors import ArgumentError, IngestError
    a = np.zeros((3, 4, 5), np.float32)
    a[1, 2, 3] = np.nan
    with pytest.raises(IngestError) as ei:
        core.grid_from_array(a)
    assert ei.value.index == (1, 2, 3)
    with pytest.raises(IngestError):
        core.grid_from_array(np.zeros((0, 3), np.float32))
    with pytest.raises(ArgumentError):
        core.grid_from_array(np.zeros((2, 2, 2, 2, 2), np.float32))
    with pytest.raises(ArgumentError):
        core.grid_from_array(np.zeros((4, 4), np.float32), (1, 1, 0, 4))
    g = core.grid_from_array(np.zeros((6, 7), np.float32))
    assert g.dims == (1, 1, 6, 7) and g.chunk_shape == (1, 1, 6, 7)


def test_tiling_order_and_flatten():
    from paper_2510_22265_b200 import core
    data = np.arange(2 * 2 * 12 * 12, dtype=np.float32).reshape(2, 2, 12, 12)
    g = core.grid_from_array(data, (1, 1, 5, 12))
    origins = [o for o, _ in core.iter_blocks(g)]
    assert origins == [(t, p, h, 0) for t in range(2) for p in range(2) for h in (0, 5, 10)]
    assert core.block_count(g.dims, g.chunk_shape) == 12
    ch = core.flatten_chunk(np.ones((2, 3, 4, 5), np.float32))
    assert ch.values.shape == (24, 5) and ch.block_shape == (2, 3, 4, 5)
    assert core.unflatten_chunk(ch.values, ch.block_shape).shape == (2, 3, 4, 5)


def test_error_stats():
    from paper_2510_22265_b200.core import error_stats
    a = np.array([0.0, 1.0, 2.0], np.float32)
    st = error_stats(a, a + np.float32(0.5))
    assert st.max_abs == 0.5 and st.rel_max == 0.25
    assert error_stats(np.ones(3), np.ones(3) + 1).rel_max == float("inf")


def test_search_budget_floor_division_matches_python():
    """budget_for_ratio uses CPython float floor division (base_codec.py:38)."""
    from oracle import oracle as o
    o.build()
    raw = 721 * 1440 * 4
    rng = np.random.default_rng(5)
    for ratio in np.concatenate([10 ** rng.uniform(0, 5.5, 500), [218576.84210526317, 1.0]]):
        assert o.budget_for_ratio(721, 1440, float(ratio)) == max(12, int(raw // float(ratio)))


# ---------------------------------------------------------------------------
# sharded assembly: world_size 2 over gloo, CPU oracle as the per-rank coder
def _oracle_records(stack):
    from oracle import oracle as o
    from paper_2510_22265_b200.container import RECORD_DTYPE
    recs = np.zeros(len(stack), RECORD_DTYPE)
    parts, offs, pos = [], [], 0
    for i, a in enumerate(stack):
        r = o.compress_chunk(a, 0.01, 1 - 1e-5)
        recs[i] = (r["mode"], 0.01, 1 - 1e-5, r["vmin"], r["vmax"], r["base_len"], r["resid_len"])
        parts.append(r["payload"])
        offs.append(pos)
        pos += len(r["payload"])
    return recs, np.frombuffer(b"".join(parts), np.uint8), np.asarray(offs, np.int64)


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    from paper_2510_22265_b200 import core, fields
    from paper_2510_22265_b200.chunk import EbccParams
    from paper_2510_22265_b200.sharding import compress_sharded
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    data = np.stack([fields.small_field("smooth", 24, 40, s) for s in range(5)])[None]
    grid = core.grid_from_array(data)
    blob = compress_sharded(grid, EbccParams(0.01), _oracle_records)
    if rank == 0:
        with open(out_path, "wb") as fh:
            fh.write(blob)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_container_equals_single_process(tmp_path):
    import socket

    import torch.multiprocessing as mp
    from oracle import oracle as o
    from paper_2510_22265_b200 import fields
    from paper_2510_22265_b200.sharding import container_offsets, shard_bounds
    o.build()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "sharded.ebcc")
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, start_method="fork")
    data = np.stack([fields.small_field("smooth", 24, 40, s) for s in range(5)])[None]
    want = o.compress(data, 0.01, 1 - 1e-5)
    got = open(out, "rb").read()
    assert got == want
    assert [shard_bounds(5, 2, r) for r in range(2)] == [(0, 3), (3, 5)]
    from paper_2510_22265_b200.container import parse
    dims, cs, recs, offs, _ = parse(got)
    sizes = recs["base_len"].astype(np.int64) + recs["resid_len"]
    np.testing.assert_array_equal(container_offsets(sizes) + 25, offs)


def test_ingest_error_precedes_shape_errors():
    """The reference scans for non-finite values before it validates the
    shape or the chunk shape (core.py:94-105): a 5-D array or a bad
    chunk_shape holding a NaN raises IngestError, not ArgumentError."""
    from paper_2510_22265_b200.core import grid_from_array
    from paper_2510_22265_b200.errors import ArgumentError, IngestError
    a = np.ones((2, 1, 1, 3, 4), np.float32)
    a[1, 0, 0, 2, 3] = np.nan
    for check in (True, False):
        with pytest.raises(IngestError):
            grid_from_array(a, check_finite=check)
        with pytest.raises(IngestError):
            grid_from_array(a[1], chunk_shape=(1, 0, 1, 1), check_finite=check)
    with pytest.raises(ArgumentError):
        grid_from_array(np.ones((2, 1, 1, 3, 4), np.float32), check_finite=False)


def test_base_codec_argument_and_container_v2_header():
    """base_codec is validated before any device work; a version-2 header
    (the opt-in J2 base layer) parses like version 1."""
    from paper_2510_22265_b200.container import VERSION_EBCOT, pack_header, parse
    from paper_2510_22265_b200.errors import ArgumentError
    from paper_2510_22265_b200.pipeline import compress_batch
    from paper_2510_22265_b200.chunk import EbccParams
    with pytest.raises(ArgumentError):
        compress_batch(np.zeros((1, 4, 4), np.float32), EbccParams(0.01), base_codec="jpeg")
    hdr = pack_header((0, 0, 0, 0), (1, 1, 1, 1), 0, VERSION_EBCOT)
    assert hdr[4:6] == b"\x02\x00"
    assert parse(hdr)[0] == (0, 0, 0, 0)
