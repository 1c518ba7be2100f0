"""ctypes binding of libebcc_gpu.so (include/ebcc_gpu.h).

There is no CPU fallback: if the library is missing or no CUDA device is
usable, every compute call raises :class:`DeviceError`.  The shared object is
built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2510_22265_b200/csrc``) so it travels with the repository snapshot.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

from .errors import (ArgumentError, DeviceError, EbccError, FormatError, IngestError,
                     ResidualInsufficient)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EBCC_LIB") or os.path.join(HERE, "libebcc_gpu.so")

OK, E_ARGUMENT, E_FORMAT, E_RESIDUAL, E_CAPACITY, E_CUDA, E_NOMEM, E_INGEST = range(8)
INPUT_ON_DEVICE = 1
OUTPUT_ON_DEVICE = 2
FULL_SEARCH = 4  # compress: every probe of the reference's searches (no candidate pruning)
CONTAINER_BODY = 8  # fetch_container: records + payloads only (one rank's span)
BASE_EBCOT = 16  # compress: the opt-in JPEG2000-style base layer ('J2'; parity unpinned)
BASE_CODECS = {"spiht": 0, "ebcot": BASE_EBCOT}

# the exported symbols include/ebcc_gpu.h declares (checked by the CPU tests)
EXPORTS = ("ebcc_abi_version", "ebcc_create", "ebcc_destroy", "ebcc_set_stream",
           "ebcc_last_error", "ebcc_last_error_index", "ebcc_compress", "ebcc_fetch_payload", "ebcc_decompress",
           "ebcc_get_stats", "ebcc_dwt", "ebcc_spiht_encode", "ebcc_spiht_decode",
           "ebcc_decode_field",
           "ebcc_selftest_div", "ebcc_fetch_container", "ebcc_host_alloc", "ebcc_host_free",
           "ebcc_error_stats", "ebcc_error_histogram", "ebcc_ssim", "ebcc_radial_spectrum",
           "ebcc_dev_probe_bench", "ebcc_parse_records", "ebcc_check_streams",
           "ebcc_host_cache_trim")


class ChunkRec(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("status", ctypes.c_int32),
                ("vmin", ctypes.c_double), ("vmax", ctypes.c_double),
                ("base_len", ctypes.c_int64), ("resid_len", ctypes.c_int64),
                ("n_base_probes", ctypes.c_int32), ("n_trunc_probes", ctypes.c_int32),
                ("resid_planes", ctypes.c_int32), ("reserved", ctypes.c_int32)]


REC_DTYPE = np.dtype([("mode", "<i4"), ("status", "<i4"), ("vmin", "<f8"), ("vmax", "<f8"),
                      ("base_len", "<i8"), ("resid_len", "<i8"), ("n_base_probes", "<i4"),
                      ("n_trunc_probes", "<i4"), ("resid_planes", "<i4"), ("reserved", "<i4")])
assert REC_DTYPE.itemsize == ctypes.sizeof(ChunkRec)


class Stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_int64), ("ms_total", ctypes.c_double),
                ("ms_encode", ctypes.c_double), ("ms_probe", ctypes.c_double),
                ("ms_other", ctypes.c_double), ("probe_launches", ctypes.c_int64),
                ("ms_probe_kernel", ctypes.c_double), ("probe_kernel_count", ctypes.c_int64),
                ("probe_kernel_fields", ctypes.c_int64), ("lanes", ctypes.c_int64),
                ("tiles_computed", ctypes.c_int64), ("tiles_probed", ctypes.c_int64)]


_lib = None
_lib_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load the shared library (raises DeviceError when it is absent)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(f"CUDA library not built: {path} (run __graft_entry__.build())")
        try:
            L = ctypes.CDLL(path)
        except OSError as exc:
            raise DeviceError(f"cannot load {path}: {exc}") from exc
        P = ctypes.c_void_p
        i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.ebcc_abi_version.restype = ctypes.c_int
        L.ebcc_create.argtypes = [i32, ctypes.POINTER(P)]
        L.ebcc_destroy.argtypes = [P]
        L.ebcc_destroy.restype = None
        L.ebcc_set_stream.argtypes = [P, P]
        L.ebcc_last_error.argtypes = [P]
        L.ebcc_last_error.restype = ctypes.c_char_p
        L.ebcc_last_error_index.argtypes = [P]
        L.ebcc_last_error_index.restype = i64
        L.ebcc_compress.argtypes = [P, P, i64, i32, i32, f64, f64, f64, f64, i32, P, P, i64, P, P]
        L.ebcc_fetch_payload.argtypes = [P, P, i64, i32]
        L.ebcc_decompress.argtypes = [P, P, P, P, i64, i32, i32, i32, i32, P]
        L.ebcc_get_stats.argtypes = [P, ctypes.POINTER(Stats)]
        L.ebcc_dwt.argtypes = [P, P, P, i64, i32, i32, i32, i32]
        L.ebcc_spiht_encode.argtypes = [P, P, i32, i32, i32, i32, P, i64, ctypes.POINTER(i64)]
        L.ebcc_spiht_decode.argtypes = [P, P, i64, i64, i32, i32, P, ctypes.POINTER(i32)]
        L.ebcc_decode_field.argtypes = [P, P, i64, i64, i32, i32, i32, P]
        L.ebcc_selftest_div.argtypes = [P, i64, ctypes.c_uint64, ctypes.POINTER(i64)]
        L.ebcc_dev_probe_bench.argtypes = [P, ctypes.c_double, i32, i32,
                                           ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_double)]
        L.ebcc_fetch_container.argtypes = [P, P, P, i64, P, i64, i32, ctypes.POINTER(i64)]
        L.ebcc_parse_records.argtypes = [P, i64, i64, P, P, ctypes.POINTER(i64),
                                         ctypes.POINTER(i32)]
        L.ebcc_check_streams.argtypes = [P, i64, P, P, i64, i32, i32, ctypes.POINTER(i32),
                                         ctypes.POINTER(i64)]
        L.ebcc_host_alloc.argtypes = [i64, ctypes.POINTER(P)]
        L.ebcc_host_free.argtypes = [P]
        L.ebcc_host_cache_trim.argtypes = []
        L.ebcc_host_cache_trim.restype = None
        L.ebcc_error_stats.argtypes = [P, P, P, i64, i64, i32, P]
        L.ebcc_error_histogram.argtypes = [P, P, P, i64, i64, i32, P, i32, P]
        L.ebcc_ssim.argtypes = [P, P, P, i64, i32, i32, i32, P]
        L.ebcc_radial_spectrum.argtypes = [P, P, i64, i32, i32, P, i32, i32, P]
        _lib = L
        return L


_PyBytes_FromStringAndSize = ctypes.pythonapi.PyBytes_FromStringAndSize
_PyBytes_FromStringAndSize.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
_PyBytes_FromStringAndSize.restype = ctypes.py_object
_PyBytes_AsString = ctypes.pythonapi.PyBytes_AsString
_PyBytes_AsString.argtypes = [ctypes.py_object]
_PyBytes_AsString.restype = ctypes.c_void_p


def _new_bytes(n: int) -> bytes:
    """A fresh, not yet shared bytes object of length n (filled by the caller
    before it is handed out, as the C API allows)."""
    return _PyBytes_FromStringAndSize(None, n)


def _bytes_ptr(b: bytes) -> int:
    return _PyBytes_AsString(b)


PINNED_MIN_BYTES = 4 << 20


def host_empty(shape, dtype) -> np.ndarray:
    """Uninitialised host array; large ones live in page-locked blocks from the
    library's cache (returned to it when the array is garbage collected), so
    the device->host copy of a result lands without a staging hop."""
    dtype = np.dtype(dtype)
    count = int(np.prod(shape, dtype=np.int64))
    nbytes = count * dtype.itemsize
    if nbytes < PINNED_MIN_BYTES:
        return np.empty(shape, dtype)
    lib = load()
    ptr = ctypes.c_void_p()
    if lib.ebcc_host_alloc(nbytes, ctypes.byref(ptr)) != OK or not ptr.value:
        raise DeviceError(f"cannot allocate {nbytes} page-locked bytes")
    buf = (ctypes.c_char * nbytes).from_address(ptr.value)
    weakref.finalize(buf, lib.ebcc_host_free, ctypes.c_void_p(ptr.value))
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)


class Context:
    """One device context (workspace + stream) of the library."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = ctypes.c_void_p()
        st = self.lib.ebcc_create(int(device), ctypes.byref(h))
        if st != OK:
            raise DeviceError(f"ebcc_create(device={device}) failed with status {st}")
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            self.lib.ebcc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def error(self) -> str:
        msg = self.lib.ebcc_last_error(self.handle)
        return msg.decode() if msg else ""

    def raise_for(self, status: int, what: str):
        if status == OK:
            return
        msg = f"{what}: {self.error()}"
        if status == E_ARGUMENT:
            raise ArgumentError(msg)
        if status == E_FORMAT:
            raise FormatError(msg)
        if status == E_RESIDUAL:
            raise ResidualInsufficient(msg)
        if status == E_INGEST:
            raise IngestError(msg, index=int(self.lib.ebcc_last_error_index(self.handle)))
        if status in (E_CUDA, E_NOMEM):
            raise DeviceError(msg)
        raise EbccError(msg)

    def stats(self) -> dict:
        s = Stats()
        self.lib.ebcc_get_stats(self.handle, ctypes.byref(s))
        return {k: getattr(s, k) for k, _ in Stats._fields_}

    def set_stream(self, stream_ptr: int):
        self.lib.ebcc_set_stream(self.handle, ctypes.c_void_p(stream_ptr))

    # -- compress ------------------------------------------------------------
    def compress(self, fields, nfields: int, rows: int, cols: int, eps_rel: float, q: float,
                 r0: float, tol: float, flags: int = 0, payload=None, payload_cap: int = 0):
        """fields: host ndarray (float32, contiguous) or device pointer (int).

        Returns (records ndarray[REC_DTYPE], offsets int64[n], total, status).
        When ``payload`` is None the payload stays in the context; fetch it
        with :meth:`fetch_payload`.
        """
        recs = np.zeros(nfields, dtype=REC_DTYPE)
        offs = np.zeros(nfields, dtype=np.int64)
        total = ctypes.c_int64(0)
        fptr = fields if isinstance(fields, int) else fields.ctypes.data
        if payload is None:
            pptr, cap = None, 0
        elif isinstance(payload, int):
            pptr, cap = payload, payload_cap
        else:
            pptr, cap = payload.ctypes.data, payload.nbytes
        st = self.lib.ebcc_compress(self.handle, ctypes.c_void_p(fptr), nfields, rows, cols,
                                    float(eps_rel), float(q), float(r0), float(tol), flags,
                                    recs.ctypes.data, pptr, cap, offs.ctypes.data,
                                    ctypes.byref(total))
        return recs, offs, int(total.value), st

    def fetch_payload(self, out, flags: int = 0):
        if isinstance(out, int):
            raise ArgumentError("pass (pointer, cap) through fetch_payload_ptr")
        st = self.lib.ebcc_fetch_payload(self.handle, out.ctypes.data, out.nbytes, flags)
        self.raise_for(st, "ebcc_fetch_payload")

    def fetch_payload_ptr(self, ptr: int, cap: int, flags: int):
        st = self.lib.ebcc_fetch_payload(self.handle, ctypes.c_void_p(ptr), cap, flags)
        self.raise_for(st, "ebcc_fetch_payload")

    def fetch_container(self, header: bytes, records: np.ndarray, payload_total: int) -> bytes:
        """The container bytes of the last compress: ``header`` (42 B) and the
        25-byte ``records`` (RECORD_DTYPE) interleaved with the payloads on the
        device, copied once into a fresh ``bytes`` object."""
        recs = np.ascontiguousarray(records)
        n = len(recs)
        size = 42 + 25 * n + int(payload_total)
        out = _new_bytes(size)
        got = ctypes.c_int64(0)
        st = self.lib.ebcc_fetch_container(self.handle, header, recs.ctypes.data if n else None,
                                           n, ctypes.c_void_p(_bytes_ptr(out)), size, 0,
                                           ctypes.byref(got))
        self.raise_for(st, "ebcc_fetch_container")
        return out

    def fetch_container_into(self, header: bytes | None, records: np.ndarray,
                             payload_total: int, ptr: int, cap: int, flags: int = 0) -> int:
        """Like :meth:`fetch_container`, into caller memory at ``ptr``;
        ``flags`` may add CONTAINER_BODY (no header).  Returns the length."""
        recs = np.ascontiguousarray(records)
        n = len(recs)
        got = ctypes.c_int64(0)
        st = self.lib.ebcc_fetch_container(self.handle, header, recs.ctypes.data if n else None,
                                           n, ctypes.c_void_p(ptr), int(cap), int(flags),
                                           ctypes.byref(got))
        self.raise_for(st, "ebcc_fetch_container")
        return int(got.value)

    # -- decompress ----------------------------------------------------------
    def decompress(self, payload, offsets: np.ndarray, recs: np.ndarray, rows: int, cols: int,
                   levels: int, out, flags: int = 0):
        pptr = payload if isinstance(payload, int) else payload.ctypes.data
        optr = out if isinstance(out, int) else out.ctypes.data
        st = self.lib.ebcc_decompress(self.handle, ctypes.c_void_p(pptr), offsets.ctypes.data,
                                      recs.ctypes.data, len(recs), rows, cols, levels, flags,
                                      ctypes.c_void_p(optr))
        self.raise_for(st, "ebcc_decompress")


    # -- unit-level entry points ---------------------------------------------
    def dwt(self, arr: np.ndarray, levels: int, inverse: bool) -> np.ndarray:
        a = np.ascontiguousarray(arr, dtype=np.float64)
        if a.ndim == 2:
            a = a[None]
        out = np.empty_like(a)
        st = self.lib.ebcc_dwt(self.handle, a.ctypes.data, out.ctypes.data, a.shape[0],
                               a.shape[1], a.shape[2], int(levels), int(inverse))
        self.raise_for(st, "ebcc_dwt")
        return out

    def spiht_encode(self, coeffs: np.ndarray, levels: int, planes: int = 24) -> bytes:
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        cap = 12 + 8 * c.size + 1024
        out = np.zeros(cap, np.uint8)
        n = ctypes.c_int64(0)
        st = self.lib.ebcc_spiht_encode(self.handle, c.ctypes.data, c.shape[0], c.shape[1],
                                        int(levels), int(planes), out.ctypes.data, cap,
                                        ctypes.byref(n))
        self.raise_for(st, "ebcc_spiht_encode")
        return out[: n.value].tobytes()

    def spiht_decode(self, data: bytes, rows: int, cols: int, prefix_len=None):
        buf = np.frombuffer(data, np.uint8).copy()
        out = np.zeros((rows, cols), np.float64)
        nl = ctypes.c_int32(0)
        st = self.lib.ebcc_spiht_decode(self.handle, buf.ctypes.data, len(buf),
                                        -1 if prefix_len is None else int(prefix_len), rows,
                                        cols, out.ctypes.data, ctypes.byref(nl))
        self.raise_for(st, "ebcc_spiht_decode")
        return out, (None if nl.value == -999 else nl.value)

    def decode_field(self, data: bytes, rows: int, cols: int, prefix_len=None,
                     midpoint: bool = True) -> np.ndarray:
        """base_codec.dequantized_field through the production inverse
        transform (the fused level kernels), float64."""
        buf = np.frombuffer(data, np.uint8).copy()
        out = np.zeros((rows, cols), np.float64)
        st = self.lib.ebcc_decode_field(self.handle, buf.ctypes.data, len(buf),
                                        -1 if prefix_len is None else int(prefix_len), rows,
                                        cols, int(bool(midpoint)), out.ctypes.data)
        self.raise_for(st, "ebcc_decode_field")
        return out


    def dev_probe_bench(self, frac: float, iters: int = 20, early: bool = False):
        """Microseconds of the level-0 kernel and of the whole full base probe
        (developer instrumentation; needs a single-lane compress first)."""
        a, b = ctypes.c_double(0), ctypes.c_double(0)
        st = self.lib.ebcc_dev_probe_bench(self.handle, float(frac), int(iters), int(early),
                                           ctypes.byref(a), ctypes.byref(b))
        self.raise_for(st, "ebcc_dev_probe_bench")
        return a.value, b.value

    def selftest_div(self, n: int, seed: int = 1) -> int:
        bad = ctypes.c_int64(0)
        st = self.lib.ebcc_selftest_div(self.handle, int(n), int(seed), ctypes.byref(bad))
        self.raise_for(st, "ebcc_selftest_div")
        return int(bad.value)


_tls = threading.local()


def context(device: int | None = None) -> Context:
    """Per-(thread, device) shared context.  Held in thread-local storage:
    when the thread exits, its contexts (and their device workspaces) are
    destroyed, so thread pools do not accumulate workspaces."""
    if device is None:
        device = int(os.environ.get("EBCC_DEVICE", "0"))
    ctxs = getattr(_tls, "contexts", None)
    if ctxs is None:
        ctxs = _tls.contexts = {}
    ctx = ctxs.get(device)
    if ctx is None:
        ctx = ctxs[device] = Context(device)
    return ctx


def trim(device: int | None = None) -> None:
    """Release this thread's context for ``device`` (all devices if None):
    its device workspaces, graphs and staging buffers; the next call
    allocates anew.  Also drops the library's cache of freed page-locked
    result blocks."""
    ctxs = getattr(_tls, "contexts", {}) or {}
    for d in list(ctxs):
        if device is None or d == device:
            ctxs.pop(d).close()
    load().ebcc_host_cache_trim()
