"""Golden values for the quality metrics (tests/golden/metrics.npz), produced
by running the reference's own ``ebcc.bench.metrics`` and ``ebcc.core`` on
seeded field pairs.  Build container only (imports /root/reference through
the scratch copy make_golden.py uses):

    python tests/golden/make_golden_metrics.py

Inputs are stored (they are small); per case the file holds the reference's
ssim, error_stats (max_abs, rel_max, rmse), error_histogram for 65 and 7 bins
and radial_power_spectrum of the reconstruction.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import REPO, import_reference  # noqa: E402

sys.path.insert(0, REPO)
from paper_2510_22265_b200 import fields  # noqa: E402


def cases(ref):
    rng = np.random.default_rng(77)
    out = []
    a = fields.small_field("smooth", 64, 96, 1)
    out.append(("noise_64x96", a, (a + rng.normal(0, 0.01, a.shape)).astype(np.float32)))
    a = fields.small_field("smooth", 100, 37, 2)
    step = float(a.max() - a.min()) / 50
    out.append(("quant_100x37", a, ref.bench.metrics.midtread_quantize(a, step)))
    a = fields.temperature_like(181, 360, seed=5, mean=250.0, std=10.0)
    out.append(("quant_181x360", a, ref.bench.metrics.midtread_quantize(a, 0.05)))
    a = fields.small_field("smooth", 33, 200, 3)
    out.append(("identical_33x200", a, a.copy()))
    a = fields.small_field("smooth", 11, 11, 4)
    out.append(("noise_11x11", a, (a + rng.normal(0, 0.1, a.shape)).astype(np.float32)))
    a = fields.precip_like(90, 120, seed=6)
    out.append(("precip_90x120", a, (a + np.abs(rng.normal(0, 1e-3, a.shape))).astype(np.float32)))
    return out


def main():
    ebcc = import_reference()
    import ebcc.bench.metrics  # noqa: F401
    store = {}
    names = []
    for name, a, b in cases(ebcc):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        m = ebcc.bench.metrics
        st = ebcc.core.error_stats(a, b)
        e65, c65 = m.error_histogram(a, b, 65)
        e7, c7 = m.error_histogram(a, b, 7)
        k, p = m.radial_power_spectrum(np.asarray(b, dtype=np.float64))
        store.update({f"{name}/a": a, f"{name}/b": b,
                      f"{name}/ssim": np.float64(m.ssim(a, b)),
                      f"{name}/stats": np.array([st.max_abs, st.rel_max, st.rmse]),
                      f"{name}/edges65": e65, f"{name}/counts65": c65,
                      f"{name}/edges7": e7, f"{name}/counts7": c7,
                      f"{name}/k": k, f"{name}/power": p})
        names.append(name)
        print(name, store[f"{name}/ssim"], st)
    store["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **store)


if __name__ == "__main__":
    main()
