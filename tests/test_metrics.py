"""Quality metrics (bench/metrics.py) on the GPU vs the reference's values.

CPU: the numpy restatement in oracle/metrics_ref.py reproduces the golden
values the reference itself produced (tests/golden/metrics.npz).
GPU: paper_2510_22265_b200.metrics reproduces them too — maxima, edges and
histogram counts exactly; sums (SSIM, RMSE, spectra) within the tolerances
below, which cover numpy's pairwise/BLAS/pocketfft summation orders.
"""

import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "metrics.npz")
SSIM_ATOL = 1e-12      # mean of O(1) terms, float64 sums in another order
RMSE_RTOL = 1e-12
SPEC_RTOL = 1e-9       # cuFFT vs pocketfft, relative to the largest bin


@pytest.fixture(scope="module")
def golden():
    z = np.load(GOLDEN)
    return z, [str(n) for n in z["names"]]


def _check_spectrum(k, p, kg, pg):
    np.testing.assert_array_equal(k, kg)
    scale = max(float(np.abs(pg).max()), 1e-300)
    assert float(np.abs(p - pg).max()) <= SPEC_RTOL * scale


def test_oracle_metrics_match_reference(golden):
    from oracle import metrics_ref as R
    z, names = golden
    for n in names:
        a, b = z[f"{n}/a"], z[f"{n}/b"]
        assert abs(R.ssim(a, b) - float(z[f"{n}/ssim"])) <= SSIM_ATOL, n
        mx, rel, rmse = R.error_stats(a, b)
        st = z[f"{n}/stats"]
        assert mx == st[0] and rel == st[1], n
        assert abs(rmse - st[2]) <= RMSE_RTOL * max(st[2], 1e-300), n
        for bins in (65, 7):
            e, c = R.error_histogram(a, b, bins)
            np.testing.assert_array_equal(e, z[f"{n}/edges{bins}"])
            np.testing.assert_array_equal(c, z[f"{n}/counts{bins}"])
        k, p = R.radial_power_spectrum(b.astype(np.float64))
        _check_spectrum(k, p, z[f"{n}/k"], z[f"{n}/power"])


@pytest.mark.gpu
def test_gpu_metrics_match_reference(golden):
    from paper_2510_22265_b200 import metrics as M
    z, names = golden
    for n in names:
        a, b = z[f"{n}/a"], z[f"{n}/b"]
        rep = M.metric_report(a, b, 1000)
        assert abs(rep.ssim - float(z[f"{n}/ssim"])) <= SSIM_ATOL, n
        assert abs(M.ssim(a, b) - rep.ssim) == 0.0
        st = z[f"{n}/stats"]
        assert rep.error_stats.max_abs == st[0] and rep.error_stats.rel_max == st[1], n
        assert abs(rep.error_stats.rmse - st[2]) <= RMSE_RTOL * max(st[2], 1e-300), n
        e, c = rep.histogram
        np.testing.assert_array_equal(e, z[f"{n}/edges65"])
        np.testing.assert_array_equal(c, z[f"{n}/counts65"])
        e7, c7 = M.error_histogram(a, b, 7)
        np.testing.assert_array_equal(e7, z[f"{n}/edges7"])
        np.testing.assert_array_equal(c7, z[f"{n}/counts7"])
        assert int(c.sum()) == a.size
        k, p = rep.spectrum
        _check_spectrum(k, p, z[f"{n}/k"], z[f"{n}/power"])
        assert rep.compression_ratio == a.size * 4 / 1000


@pytest.mark.gpu
def test_gpu_metrics_batch_full_size_vs_oracle():
    """A stack of 721x1440 pairs (bench shape): batched reports equal the
    single-field ones, and agree with the restatement."""
    from oracle import metrics_ref as R
    from paper_2510_22265_b200 import fields
    from paper_2510_22265_b200 import metrics as M
    rng = np.random.default_rng(9)
    a = np.stack([fields.temperature_like(721, 1440, seed=40 + i, mean=250.0, std=12.0)
                  for i in range(3)])
    b = (a + rng.normal(0, 0.05, a.shape)).astype(np.float32)
    b[1] = a[1]  # an identical pair
    reps = M.metric_reports(a, b, [1 << 20, 1 << 21, 1 << 22])
    for i in range(3):
        one = M.metric_report(a[i], b[i], [1 << 20, 1 << 21, 1 << 22][i])
        assert one.ssim == reps[i].ssim
        np.testing.assert_array_equal(one.histogram[1], reps[i].histogram[1])
        _check_spectrum(one.spectrum[0], one.spectrum[1], reps[i].spectrum[0], reps[i].spectrum[1])
        assert abs(reps[i].ssim - R.ssim(a[i], b[i])) <= 1e-11
        e, c = R.error_histogram(a[i], b[i], 65)
        np.testing.assert_array_equal(reps[i].histogram[0], e)
        np.testing.assert_array_equal(reps[i].histogram[1], c)
        mx, rel, rmse = R.error_stats(a[i], b[i])
        assert reps[i].error_stats.max_abs == mx and reps[i].error_stats.rel_max == rel
        assert abs(reps[i].error_stats.rmse - rmse) <= 1e-11 * max(rmse, 1e-300)
        k, p = R.radial_power_spectrum(b[i].astype(np.float64))
        _check_spectrum(reps[i].spectrum[0], reps[i].spectrum[1], k, p)
    assert reps[1].ssim == 1.0


def test_metrics_argument_errors_without_gpu():
    from paper_2510_22265_b200 import metrics as M
    from paper_2510_22265_b200.errors import ArgumentError
    with pytest.raises(ArgumentError):
        M.ssim(np.zeros((12, 12), np.float32), np.zeros((12, 13), np.float32))
    with pytest.raises(ArgumentError):
        M.error_histogram(np.zeros(5), np.zeros(5), bins=0)
    with pytest.raises(ArgumentError):
        M.radial_power_spectrum(np.zeros((2, 3, 4)))
