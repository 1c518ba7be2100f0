"""ctypes front end of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Loads oracle/libebcc_oracle.so (built by ``make -C oracle`` or by
``__graft_entry__.build()``).  Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs import this module; the product package never
does.  Grid-level helpers reuse the product's host container/tiling code so
that oracle containers are assembled exactly like product containers.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libebcc_oracle.so")

_lib = None


class ChunkResult(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("status", ctypes.c_int32),
                ("vmin", ctypes.c_double), ("vmax", ctypes.c_double),
                ("base_len", ctypes.c_int64), ("resid_len", ctypes.c_int64),
                ("n_base_probes", ctypes.c_int32), ("n_trunc_probes", ctypes.c_int32),
                ("resid_planes", ctypes.c_int32), ("pad", ctypes.c_int32)]


def build(force: bool = False) -> str:
    srcs = [os.path.join(HERE, f) for f in ("ebcc_oracle.c", "ebcot_oracle.c", "ebcc_oracle.h")]
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < max(os.path.getmtime(f) for f in srcs):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i32, i64, f64 = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        L.eo_default_levels.argtypes = [i32, i32]
        L.eo_clamp_levels.argtypes = [i32, i32, i32]
        L.eo_forward_dwt.argtypes = [P, i32, i32, i32]
        L.eo_inverse_dwt.argtypes = [P, i32, i32, i32]
        L.eo_spiht_encode.argtypes = [P, i32, i32, i32, i64, i32, P, i64]
        L.eo_spiht_encode.restype = i64
        L.eo_spiht_decode.argtypes = [P, i64, i64, i32, i32, P, P]
        L.eo_budget_for_ratio.argtypes = [i32, i32, f64]
        L.eo_budget_for_ratio.restype = i64
        L.eo_compress_chunk.argtypes = [P, i32, i32, f64, f64, f64, f64, P, P, i64, P, P, i32,
                                        P, i32]
        L.eo_decompress_chunk.argtypes = [i32, f64, f64, P, i64, i64, i32, i32, P]
        L.eo_base_encode_budget.argtypes = [P, i32, i32, i64, f64, P, i64, P, P]
        L.eo_base_encode_budget.restype = i64
        L.eo_set_base_codec.argtypes = [i32]
        L.eo_ebcot_blocks.argtypes = [i32, i32, i32, P, i32]
        L.eo_ebcot_encode.argtypes = [P, i32, i32, i32, i64, P, i64]
        L.eo_ebcot_encode.restype = i64
        L.eo_ebcot_decode.argtypes = [P, i64, i32, i32, P]
        L.eo_mq_encode.argtypes = [P, P, i64, P]
        L.eo_mq_encode.restype = i64
        L.eo_mq_decode.argtypes = [P, i64, P, i64, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def default_levels(rows, cols):
    return lib().eo_default_levels(rows, cols)


def forward_dwt(x, levels=None):
    a = np.array(x, dtype=np.float64, copy=True, order="C")
    r, c = a.shape
    if levels is None:
        levels = default_levels(r, c)
    levels = lib().eo_clamp_levels(r, c, levels)
    lib().eo_forward_dwt(_p(a), r, c, levels)
    return a, levels


def inverse_dwt(coeffs, levels):
    a = np.array(coeffs, dtype=np.float64, copy=True, order="C")
    lib().eo_inverse_dwt(_p(a), a.shape[0], a.shape[1], levels)
    return a


def spiht_encode(coeffs, levels, max_bytes=None, planes=24) -> bytes:
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    cap = 12 + 40 * c.size + 64
    out = np.zeros(cap, np.uint8)
    n = lib().eo_spiht_encode(_p(c), c.shape[0], c.shape[1], levels,
                              -1 if max_bytes is None else int(max_bytes), planes, _p(out), cap)
    if n < 0:
        raise RuntimeError(f"oracle encode failed ({-n})")
    return out[:n].tobytes()


def decode_with_plane(data: bytes, rows, cols, prefix_len=None):
    buf = np.frombuffer(data, np.uint8).copy()
    out = np.zeros(rows * cols, np.float64)
    nl = ctypes.c_int(0)
    st = lib().eo_spiht_decode(_p(buf), len(buf), -1 if prefix_len is None else int(prefix_len),
                               rows, cols, _p(out), ctypes.byref(nl))
    if st:
        raise RuntimeError(f"oracle decode failed ({st})")
    return out.reshape(rows, cols), (None if nl.value == -999 else nl.value)


# ---- opt-in JPEG2000-style base layer (parity unpinned: no reference) ----
BASE_CODECS = {"spiht": 0, "ebcot": 1}


def mq_encode(bits, cx) -> bytes:
    b = np.ascontiguousarray(bits, np.uint8)
    c = np.ascontiguousarray(cx, np.uint8)
    out = np.zeros(2 * b.size + 16, np.uint8)
    n = lib().eo_mq_encode(_p(b), _p(c), b.size, _p(out))
    return out[:n].tobytes()


def mq_decode(data: bytes, cx) -> np.ndarray:
    c = np.ascontiguousarray(cx, np.uint8)
    buf = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
    out = np.zeros(c.size, np.uint8)
    lib().eo_mq_decode(_p(buf), len(data), _p(c), c.size, _p(out))
    return out


def ebcot_blocks(rows, cols, levels) -> np.ndarray:
    n = lib().eo_ebcot_blocks(rows, cols, levels, None, 0)
    out = np.zeros((max(n, 1), 5), np.int32)
    lib().eo_ebcot_blocks(rows, cols, levels, _p(out), n)
    return out[:n]


def ebcot_encode(coeffs, levels, max_bytes=None) -> bytes:
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    cap = 12 + 8 * c.size + 4096
    out = np.zeros(cap, np.uint8)
    n = lib().eo_ebcot_encode(_p(c), c.shape[0], c.shape[1], levels,
                              -1 if max_bytes is None else int(max_bytes), _p(out), cap)
    if n < 0:
        raise RuntimeError(f"oracle ebcot encode failed ({-n})")
    return out[:n].tobytes()


def ebcot_decode(data: bytes, rows, cols) -> np.ndarray:
    buf = np.frombuffer(data, np.uint8).copy()
    out = np.zeros(rows * cols, np.float64)
    st = lib().eo_ebcot_decode(_p(buf), len(buf), rows, cols, _p(out))
    if st:
        raise RuntimeError(f"oracle ebcot decode failed ({st})")
    return out.reshape(rows, cols)


def budget_for_ratio(rows, cols, ratio):
    return lib().eo_budget_for_ratio(rows, cols, float(ratio))


def compress_chunk(values, eps_rel, q=1 - 1e-5, r0=10.0, tol=1e-3, trace=False,
                   base_codec="spiht"):
    """Compress one 2D float32 chunk; returns a dict (payload bytes, record
    fields, probe traces when ``trace``)."""
    lib().eo_set_base_codec(BASE_CODECS[base_codec])
    v = np.ascontiguousarray(values, dtype=np.float32)
    rows, cols = v.shape
    cap = 16 * v.size + 1024
    pay = np.zeros(cap, np.uint8)
    res = ChunkResult()
    tcap = 4096
    tb = np.zeros(tcap, np.int64)
    tq = np.zeros(tcap, np.float64)
    tt = np.zeros(tcap, np.int64)
    st = lib().eo_compress_chunk(_p(v), rows, cols, float(eps_rel), float(q), float(r0),
                                 float(tol), ctypes.byref(res), _p(pay), cap,
                                 _p(tb) if trace else None, _p(tq) if trace else None, tcap,
                                 _p(tt) if trace else None, tcap)
    lib().eo_set_base_codec(0)
    out = {"status": st, "mode": res.mode, "vmin": res.vmin, "vmax": res.vmax,
           "base_len": res.base_len, "resid_len": res.resid_len,
           "n_base_probes": res.n_base_probes, "n_trunc_probes": res.n_trunc_probes,
           "resid_planes": res.resid_planes,
           "payload": pay[: res.base_len + res.resid_len].tobytes() if st == 0 else b""}
    if trace:
        nb = min(res.n_base_probes, tcap)
        out["base_trace"] = [(int(tb[i]), float(tq[i])) for i in range(nb)]
        out["trunc_trace"] = [int(tt[i]) for i in range(min(res.n_trunc_probes, tcap))]
    return out


def decompress_chunk(mode, vmin, vmax, payload: bytes, base_len, resid_len, rows, cols):
    buf = np.frombuffer(payload, np.uint8).copy() if payload else np.zeros(1, np.uint8)
    out = np.zeros(rows * cols, np.float32)
    st = lib().eo_decompress_chunk(int(mode), float(vmin), float(vmax), _p(buf), int(base_len),
                                   int(resid_len), rows, cols, _p(out))
    if st:
        raise RuntimeError(f"oracle decompress failed ({st})")
    return out.reshape(rows, cols)


STATUS_NAMES = {1: "ArgumentError", 2: "FormatError", 3: "ResidualInsufficient"}


def compress(array, rel_error=0.01, q=1 - 1e-5, chunk_shape=None,
             base_codec="spiht") -> bytes:
    """Oracle equivalent of the reference api.compress (container bytes);
    ``base_codec="ebcot"``: the opt-in JPEG2000-style base layer (container
    version 2)."""
    from paper_2510_22265_b200 import core
    from paper_2510_22265_b200.chunk import CompressedChunk, Mode
    from paper_2510_22265_b200.container import write_bytes
    from paper_2510_22265_b200 import errors
    grid = core.grid_from_array(np.asarray(array), chunk_shape)
    chunks = []
    for origin, block in core.iter_blocks(grid):
        ch = core.flatten_chunk(block, origin)
        r = compress_chunk(ch.values, rel_error, q, base_codec=base_codec)
        if r["status"]:
            cls = getattr(errors, STATUS_NAMES.get(r["status"], "EbccError"))
            raise cls(f"chunk at origin {origin}: oracle status {r['status']}")
        chunks.append(CompressedChunk(mode=Mode(r["mode"]), epsilon_rel=rel_error, q=q,
                                      vmin=r["vmin"], vmax=r["vmax"], base_len=r["base_len"],
                                      residual_len=r["resid_len"], payload=r["payload"],
                                      rows=ch.rows, cols=ch.cols, block_shape=ch.block_shape,
                                      origin=origin))
    return write_bytes(chunks, grid.dims, grid.chunk_shape,
                       version=2 if base_codec == "ebcot" else 1)


def decompress(buf: bytes) -> np.ndarray:
    from paper_2510_22265_b200.container import read_file
    chunks, dims, _ = read_file(buf)
    out = np.empty(tuple(dims), np.float32)
    for cc in chunks:
        v = decompress_chunk(cc.mode, cc.vmin, cc.vmax, cc.payload, cc.base_len,
                             cc.residual_len, cc.rows, cc.cols)
        t0, p0, h0, w0 = cc.origin
        t, p, h, w = cc.block_shape
        out[t0:t0 + t, p0:p0 + p, h0:h0 + h, w0:w0 + w] = v.reshape(t, p, h, w)
    return out
