"""CPU restatement of the reference's quality metrics — TEST INFRASTRUCTURE.

Only tests/ may import this module: it is the checker for the GPU metrics in
``paper_2510_22265_b200/metrics.py`` (csrc/metrics.cu), never a product path.
Each function restates ``pkg/src/ebcc/bench/metrics.py`` (numpy, float64) at
the cited lines; it is pinned against values produced by the reference
itself (tests/golden/metrics.npz, tests/golden/make_golden_metrics.py).
"""

from __future__ import annotations

import numpy as np

WINDOW, SIGMA, K1, K2, FLOOR = 11, 1.5, 0.01, 0.03, 1e-30  # metrics.py:13-17


def gaussian_kernel() -> np.ndarray:
    # metrics.py:31-35
    half = WINDOW // 2
    x = np.arange(-half, half + 1, dtype=np.float64)
    k = np.exp(-(x * x) / (2.0 * SIGMA ** 2))
    return k / k.sum()


def _valid_filter(img: np.ndarray, k: np.ndarray) -> np.ndarray:
    # metrics.py:38-44: separable correlation, valid region, rows then columns
    w = k.size
    r, c = img.shape
    h = np.zeros((r, c - w + 1))
    for t in range(w):
        h += img[:, t:t + c - w + 1] * k[t]
    v = np.zeros((r - w + 1, c - w + 1))
    for t in range(w):
        v += h[t:t + r - w + 1, :] * k[t]
    return v


def ssim(a, b) -> float:
    # metrics.py:47-75
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if np.array_equal(a, b):
        return 1.0
    rng = max(float(a.max() - a.min()), FLOOR)
    c1, c2 = (K1 * rng) ** 2, (K2 * rng) ** 2
    k = gaussian_kernel()
    mu_a, mu_b = _valid_filter(a, k), _valid_filter(b, k)
    mu_aa, mu_bb, mu_ab = mu_a * mu_a, mu_b * mu_b, mu_a * mu_b
    var_a = _valid_filter(a * a, k) - mu_aa
    var_b = _valid_filter(b * b, k) - mu_bb
    cov = _valid_filter(a * b, k) - mu_ab
    num = (2.0 * mu_ab + c1) * (2.0 * cov + c2)
    den = (mu_aa + mu_bb + c1) * (var_a + var_b + c2)
    return float(np.mean(num / den))


def error_histogram(a, b, bins: int = 65):
    # metrics.py:78-99: edges from the largest |error|, last bin closed
    diff = (np.asarray(b, np.float64) - np.asarray(a, np.float64)).ravel()
    span = float(np.abs(diff).max())
    if span == 0.0:
        span = FLOOR
    edges = np.linspace(-span, span, bins + 1)
    k = np.searchsorted(edges, diff, side="right") - 1
    k[diff == edges[-1]] = bins - 1
    ok = (k >= 0) & (k < bins)
    return edges, np.bincount(k[ok], minlength=bins)[:bins]


def radial_power_spectrum(a):
    # metrics.py:102-125
    a = np.asarray(a, dtype=np.float64)
    rows, cols = a.shape
    power = np.abs(np.fft.fft2(a) / (rows * cols)) ** 2
    k1 = np.fft.fftfreq(rows) * rows
    k2 = np.fft.fftfreq(cols) * cols
    m = min(rows, cols)
    kr = np.hypot(k1[:, None] * (m / rows), k2[None, :] * (m / cols))
    kmax = m // 2
    idx = np.rint(kr).astype(np.int64)
    ok = (idx >= 1) & (idx <= kmax)
    return np.arange(1, kmax + 1), np.bincount(idx[ok], weights=power[ok], minlength=kmax + 1)[1:]


def error_stats(a, b):
    # core.py:189-207
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.abs(b - a)
    mx = float(d.max())
    span = float(a.max() - a.min())
    rel = mx / span if span > 0 else (0.0 if mx == 0.0 else float("inf"))
    return mx, rel, float(np.sqrt(np.mean(d * d)))
