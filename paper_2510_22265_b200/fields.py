"""Seeded synthetic stand-ins for the ERA5 fields named in BASELINE.json.

ERA5 itself is not available offline; these generators reproduce the shapes
and value distributions of the five BASELINE.json configurations (SURVEY.md
§8(d)).  Every field is a Gaussian random field with an isotropic power-law
spectrum drawn from ``numpy.random.default_rng(seed)`` and synthesised with an
inverse FFT, then standardised and rescaled.  Generation is never timed.

The spectral convention (DC bin pinned to 1 before the power law, complex
normal spectrum, real part of the inverse FFT, zero-mean unit-variance
standardisation) follows the reference's synthetic-field generator
(pkg/src/ebcc/bench/fields.py:30-41) so the fields have the same statistics.
"""

from __future__ import annotations

import numpy as np

GRID_025 = (721, 1440)       # 0.25 degree global lat-lon
GRID_0625 = (2881, 5760)     # 1/16 degree global lat-lon


def power_law_grf(rows: int, cols: int, seed: int, beta: float) -> np.ndarray:
    """Unit-variance float64 GRF whose power spectrum falls as k**-beta."""
    gen = np.random.default_rng(seed)
    fy = np.fft.fftfreq(rows).reshape(rows, 1)
    fx = np.fft.fftfreq(cols).reshape(1, cols)
    kmag = np.hypot(fy, fx)
    kmag[0, 0] = 1.0
    amp = np.power(kmag, -0.5 * beta)
    re = gen.standard_normal((rows, cols))
    im = gen.standard_normal((rows, cols))
    g = np.fft.ifft2((re + 1j * im) * amp).real
    g = g - g.mean()
    sd = g.std()
    return g / sd if sd > 0 else g


def temperature_like(rows: int, cols: int, seed: int = 0, mean: float = 280.0,
                     std: float = 15.0, beta: float = 3.0) -> np.ndarray:
    """Config 1: smooth k^-3 field rescaled to (mean, std), float32."""
    return (power_law_grf(rows, cols, seed, beta) * std + mean).astype(np.float32)


def precip_like(rows: int, cols: int, seed: int, beta: float = 2.5,
                dry_percentile: float = 60.0) -> np.ndarray:
    """Config 3: exp of a k^-2.5 GRF with the lowest 60% set to zero."""
    f = np.exp(power_law_grf(rows, cols, seed, beta))
    cut = np.percentile(f, dry_percentile)
    f[f < cut] = 0.0
    return f.astype(np.float32)


def config1_field() -> np.ndarray:
    """Single 721x1440 temperature-like field (BASELINE.json configs[0])."""
    return temperature_like(*GRID_025, seed=0)


def config2_levels(levels: int = 37, rows: int = GRID_025[0],
                   cols: int = GRID_025[1]) -> np.ndarray:
    """37 independent k^-3 levels, mean 200..300, std 2..20 (configs[1]).

    Returns (1, levels, rows, cols) float32.
    """
    out = np.empty((1, levels, rows, cols), dtype=np.float32)
    for lev in range(levels):
        frac = lev / max(1, levels - 1)
        out[0, lev] = temperature_like(rows, cols, seed=1000 + lev,
                                       mean=200.0 + 100.0 * frac,
                                       std=2.0 + 18.0 * frac)
    return out


def config3_precip(steps: int = 24, rows: int = GRID_025[0],
                   cols: int = GRID_025[1]) -> np.ndarray:
    """24 precipitation-like time steps, (steps, 1, rows, cols) (configs[2])."""
    out = np.empty((steps, 1, rows, cols), dtype=np.float32)
    for t in range(steps):
        out[t, 0] = precip_like(rows, cols, seed=2000 + t)
    return out


def config4_field(v: int, rows: int = GRID_0625[0], cols: int = GRID_0625[1]) -> np.ndarray:
    """Variable v of configs[3]: 0-5 smooth k^-3, 6-9 wind-like k^-5/3."""
    gen = np.random.default_rng(3000 + v)
    if v < 6:
        mean = float(gen.uniform(0.0, 300.0))
        std = float(gen.uniform(1.0, 20.0))
        return temperature_like(rows, cols, seed=3000 + v, mean=mean, std=std)
    return temperature_like(rows, cols, seed=3000 + v, mean=0.0, std=10.0, beta=5.0 / 3.0)


def config4_fields(nvars: int = 10, rows: int = GRID_0625[0],
                   cols: int = GRID_0625[1]):
    """Ten 2881x5760 variables: 6 smooth k^-3 + 4 wind-like k^-5/3 (configs[3]).

    Yields (var_index, float32 field) so callers never hold all of them.
    """
    for v in range(nvars):
        yield v, config4_field(v, rows, cols)


def config5_field(field_id: int, rows: int = GRID_025[0],
                  cols: int = GRID_025[1]) -> np.ndarray:
    """One field of the 8 var x 37 level x 8 step sweep (configs[4])."""
    gen = np.random.default_rng(4000 + field_id)
    mean = float(gen.uniform(200.0, 300.0))
    std = float(gen.uniform(2.0, 20.0))
    return temperature_like(rows, cols, seed=4000 + field_id, mean=mean, std=std)


CONFIG5_FIELDS = 8 * 37 * 8


_C5_SHARED = None  # (buffer, shape, ids) inherited by the fork pool's workers


def _fill_config5(lo_hi):
    buf, shape, ids = _C5_SHARED
    out = np.frombuffer(buf, dtype=np.float32).reshape(shape)
    for k in range(*lo_hi):
        out[k] = config5_field(int(ids[k]), shape[1], shape[2])
    return lo_hi[1] - lo_hi[0]


def config5_stack(ids, rows: int = GRID_025[0], cols: int = GRID_025[1],
                  workers: int = 0) -> np.ndarray:
    """Fields ``ids`` of the configs[4] sweep as one (len(ids), rows, cols)
    float32 array, generated by a fork pool into shared anonymous memory (the
    2,368-field sweep is 9.8 GB; one core needs ~2 min for it).  Every field
    is byte-identical to ``config5_field(id)``."""
    import mmap
    import multiprocessing as mp
    import os

    global _C5_SHARED
    ids = np.asarray(ids, dtype=np.int64)
    n = len(ids)
    shape = (n, rows, cols)
    buf = mmap.mmap(-1, max(1, n * rows * cols * 4))  # MAP_SHARED|MAP_ANONYMOUS
    cores = max(1, min(workers or len(os.sched_getaffinity(0)), n))
    _C5_SHARED = (buf, shape, ids)
    try:
        if cores == 1:
            _fill_config5((0, n))
        else:
            step = max(1, -(-n // (cores * 4)))
            with mp.get_context("fork").Pool(cores) as pool:
                pool.map(_fill_config5, [(lo, min(n, lo + step)) for lo in range(0, n, step)])
    finally:
        _C5_SHARED = None
    return np.frombuffer(buf, dtype=np.float32, count=n * rows * cols).reshape(shape)


def vortex_like(rows: int, cols: int, seed: int) -> np.ndarray:
    """Wind-speed-like field: the speed of a superposition of a few Gaussian
    point vortices (random centres, radii, signed circulations) on a weak
    k^-3 background; sharp cores and smooth far fields."""
    gen = np.random.default_rng(seed)
    y, x = np.mgrid[0:rows, 0:cols].astype(np.float64)
    u = np.zeros((rows, cols))
    v = np.zeros((rows, cols))
    for _ in range(int(gen.integers(2, 6))):
        y0, x0 = gen.uniform(0, rows), gen.uniform(0, cols)
        rad = gen.uniform(0.05, 0.3) * max(rows, cols)
        circ = gen.choice([-1.0, 1.0]) * gen.uniform(5.0, 30.0)
        w = circ * np.exp(-((y - y0) ** 2 + (x - x0) ** 2) / (2.0 * rad * rad)) / rad
        u -= w * (y - y0)
        v += w * (x - x0)
    speed = np.hypot(u, v) + 0.5 * power_law_grf(rows, cols, seed + 104729, 3.0)
    return speed.astype(np.float32)


def small_field(kind: str, rows: int, cols: int, seed: int) -> np.ndarray:
    """Small test fields: 'smooth', 'spiky' (isolated heavy-tailed outliers),
    'precip' (intermittent), 'vortex' (point-vortex wind speed), 'noise'
    (white) — float32."""
    if kind == "smooth":
        return temperature_like(rows, cols, seed=seed, mean=0.0, std=1.0)
    if kind == "precip":
        return precip_like(rows, cols, seed=seed)
    if kind == "vortex":
        return vortex_like(rows, cols, seed)
    if kind == "noise":
        return np.random.default_rng(seed).standard_normal((rows, cols)).astype(np.float32)
    if kind == "spiky":
        f = power_law_grf(rows, cols, seed, 3.0)
        gen = np.random.default_rng(seed + 7919)
        n = rows * cols
        k = max(1, n // 4000)
        at = gen.choice(n, size=k, replace=False)
        f.reshape(-1)[at] += gen.choice([-1.0, 1.0], size=k) * np.exp(gen.normal(2.0, 0.7, size=k))
        return f.astype(np.float32)
    raise ValueError(f"unknown kind {kind!r}")
