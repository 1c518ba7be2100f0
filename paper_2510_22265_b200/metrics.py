"""Quality metrics of the reference's benchmark harness, computed on the GPU.

Mirrors ``pkg/src/ebcc/bench/metrics.py`` (same names, arguments, return
values and ``ArgumentError`` cases) on top of the device kernels in
``csrc/metrics.cu``:

* ``ssim``                   metrics.py:47-75  (mean SSIM, 11x11 Gaussian, sigma 1.5)
* ``error_histogram``        metrics.py:78-99  (symmetric bins, exact counts)
* ``radial_power_spectrum``  metrics.py:102-125 (cuFFT + annulus sums)
* ``metric_report``          metrics.py:176-186, plus ``metric_reports`` for a
  batch of same-shape fields in one device call per metric.

Everything is float64 like the reference; sums run in a fixed order on the
device, so SSIM / RMSE / spectra agree with numpy to the last few bits (the
parity tests state the tolerances) while maxima and histogram counts are
exact.  There is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .core import ErrorStats
from .errors import ArgumentError

SSIM_WINDOW = 11
_RANGE_FLOOR = 1e-30


@dataclass(frozen=True)
class MetricReport:
    """Quality summary for one original/reconstruction pair (metrics.py:20-28)."""

    error_stats: ErrorStats
    ssim: float
    histogram: tuple  # (bin edges, counts)
    spectrum: tuple  # (wavenumbers, power)
    compression_ratio: float


def _stack(a, name="a") -> np.ndarray:
    """(n, rows, cols) float32, C-contiguous."""
    x = np.ascontiguousarray(np.asarray(a), dtype=np.float32)
    if x.ndim == 2:
        x = x[None]
    if x.ndim != 3:
        raise ArgumentError(f"{name}: expected 2D fields or a stack of them, got {x.shape}")
    return x


def _pair(a, b):
    aa, bb = np.asarray(a), np.asarray(b)
    if aa.shape != bb.shape:
        raise ArgumentError(f"shape mismatch: {aa.shape} vs {bb.shape}")
    return _stack(aa, "a"), _stack(bb, "b")


def _call(name, *args):
    ctx = _lib.context()
    st = getattr(ctx.lib, name)(ctx.handle, *args)
    ctx.raise_for(st, name)


def _raw_stats(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    n, r, c = a.shape
    out = np.zeros((n, 5), np.float64)
    _call("ebcc_error_stats", a.ctypes.data, b.ctypes.data, n, r * c, 0, out.ctypes.data)
    return out


def _stats_from_raw(raw, npoints) -> ErrorStats:
    """core.error_stats (core.py:189-207) from the device reductions."""
    max_abs, lo, hi, sumsq = float(raw[0]), float(raw[1]), float(raw[2]), float(raw[3])
    span = hi - lo
    if span > 0.0:
        rel = max_abs / span
    else:
        rel = 0.0 if max_abs == 0.0 else float("inf")
    return ErrorStats(max_abs=max_abs, rel_max=rel, rmse=float(np.sqrt(sumsq / npoints)))


def error_stats_batch(originals, reconstructions) -> list:
    """``core.error_stats`` for each field of a stack, on the device."""
    a, b = _pair(originals, reconstructions)
    raw = _raw_stats(a, b)
    return [_stats_from_raw(raw[i], a.shape[1] * a.shape[2]) for i in range(len(a))]


def _edges_for(max_abs: float, bins: int) -> np.ndarray:
    span = float(max_abs)
    if span == 0.0:
        span = _RANGE_FLOOR
    return np.linspace(-span, span, bins + 1)


def _histograms(a, b, bins, raw) -> list:
    n, r, c = a.shape
    edges = np.stack([_edges_for(raw[i, 0], bins) for i in range(n)])
    counts = np.zeros((n, bins), np.int64)
    _call("ebcc_error_histogram", a.ctypes.data, b.ctypes.data, n, r * c, bins,
          np.ascontiguousarray(edges).ctypes.data, 0, counts.ctypes.data)
    return [(edges[i], counts[i]) for i in range(n)]


def error_histogram(a, b, bins: int = 65):
    """Histogram of point-wise errors in symmetric bins centered on zero.

    Returns (edges, counts); counts always sum to the element count.
    """
    if np.asarray(a).shape != np.asarray(b).shape:
        raise ArgumentError(f"shape mismatch: {np.asarray(a).shape} vs {np.asarray(b).shape}")
    if bins < 1:
        raise ArgumentError("bins must be >= 1")
    aa = np.asarray(a, dtype=np.float32).reshape(1, 1, -1)
    bb = np.asarray(b, dtype=np.float32).reshape(1, 1, -1)
    aa, bb = _stack(aa[0], "a"), _stack(bb[0], "b")
    return _histograms(aa, bb, int(bins), _raw_stats(aa, bb))[0]


def _ssims(a, b) -> np.ndarray:
    n, r, c = a.shape
    if min(r, c) < SSIM_WINDOW:
        raise ArgumentError(f"fields must be at least {SSIM_WINDOW}x{SSIM_WINDOW}")
    out = np.zeros(n, np.float64)
    _call("ebcc_ssim", a.ctypes.data, b.ctypes.data, n, r, c, 0, out.ctypes.data)
    return out


def ssim(a, b) -> float:
    """Mean local structural similarity (11x11 Gaussian window, sigma 1.5).

    The dynamic range is taken from the first argument; identical inputs
    with zero range score 1.
    """
    aa, bb = _pair(a, b)
    if aa.shape[0] != 1:
        raise ArgumentError("ssim compares one 2D field pair; use metric_reports for stacks")
    return float(_ssims(aa, bb)[0])


@lru_cache(maxsize=16)
def _wavenumber_map(rows: int, cols: int):
    # metrics.py:112-121: integer wavenumbers scaled to the min-extent domain
    k1 = np.fft.fftfreq(rows) * rows
    k2 = np.fft.fftfreq(cols) * cols
    m = min(rows, cols)
    kr = np.hypot(k1[:, None] * (m / rows), k2[None, :] * (m / cols))
    kmax = m // 2
    idx = np.rint(kr).astype(np.int64)
    idx[(idx < 1) | (idx > kmax)] = -1
    return np.ascontiguousarray(idx.astype(np.int32)), kmax


def _spectra(x: np.ndarray) -> list:
    n, r, c = x.shape
    idx, kmax = _wavenumber_map(r, c)
    if kmax < 1:
        return [(np.arange(1, kmax + 1), np.zeros(0)) for _ in range(n)]
    out = np.zeros((n, kmax), np.float64)
    _call("ebcc_radial_spectrum", x.ctypes.data, n, r, c, idx.ctypes.data, kmax, 0,
          out.ctypes.data)
    return [(np.arange(1, kmax + 1), out[i]) for i in range(n)]


def radial_power_spectrum(a):
    """Isotropic power spectrum: periodogram energy summed in integer
    wavenumber annuli (1 .. floor(min(rows, cols)/2)), DC excluded."""
    x = np.asarray(a)
    if x.ndim != 2:
        raise ArgumentError(f"expected a 2D field, got {x.shape}")
    return _spectra(_stack(x))[0]


def metric_reports(originals, reconstructions, compressed_bytes, bins: int = 65) -> list:
    """``metric_report`` for every field of a (n, rows, cols) stack: one
    device call per metric for the whole stack."""
    a, b = _pair(originals, reconstructions)
    if bins < 1:
        raise ArgumentError("bins must be >= 1")
    sizes = np.broadcast_to(np.asarray(compressed_bytes, dtype=np.int64), (len(a),))
    raw = _raw_stats(a, b)
    npts = a.shape[1] * a.shape[2]
    hists = _histograms(a, b, int(bins), raw)
    ss = _ssims(a, b)
    spec = _spectra(b)
    return [MetricReport(error_stats=_stats_from_raw(raw[i], npts), ssim=float(ss[i]),
                         histogram=hists[i], spectrum=spec[i],
                         compression_ratio=float(npts * 4 / max(int(sizes[i]), 1)))
            for i in range(len(a))]


def metric_report(original, reconstructed, compressed_bytes: int,
                  bins: int = 65) -> MetricReport:
    """Full quality summary for one pair plus the achieved ratio."""
    aa, bb = np.asarray(original), np.asarray(reconstructed)
    if aa.ndim != 2:
        raise ArgumentError(f"expected a 2D field, got {aa.shape}")
    return metric_reports(aa, bb, compressed_bytes, bins)[0]
