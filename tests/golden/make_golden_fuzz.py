"""Fixtures for the reference's acceptance fuzz distribution, run through the
unmodified reference (round 2).

Generates (in this container only; the reference does not travel):

* fuzz.json — the error-bound fuzz of pkg/tests/test_acceptance.py:48-80
  re-created with THIS repo's generators: 1000 chunks, the same forced corner
  shapes then log-uniform shapes in 8..256 (numpy default_rng(2024)), kinds
  cycling smooth / vortex / spiky, eps cycling (0.001, 0.005, 0.01, 0.05,
  0.10), q cycling over (1-1e-3, 1-1e-4, 1-1e-5, 1-1e-6, 1.0) every 5 cases,
  seed = case index.  Per case: the reference's container SHA-256 and length.
* edge.json — signed zeros at the minimum, and a custom r0 whose first budget
  needs CPython float floor division (4152960 // 218576.84210526317 == 18,
  floor of the quotient is 19; base_codec.py:38).
"""
from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from make_golden import import_reference  # noqa: E402
from paper_2510_22265_b200 import fields  # noqa: E402

EPS_GRID = (0.001, 0.005, 0.01, 0.05, 0.10)
Q_GRID = (1 - 1e-3, 1 - 1e-4, 1 - 1e-5, 1 - 1e-6, 1.0)
KINDS = ("smooth", "vortex", "spiky")
FORCED = [(8, 8), (256, 256), (8, 256), (255, 17), (33, 129)]


def fuzz_cases(total=1000):
    rng = np.random.default_rng(2024)
    cases = []
    for i in range(total):
        if i < len(FORCED):
            rows, cols = FORCED[i]
        else:
            rows = int(np.exp(rng.uniform(np.log(8), np.log(256))))
            cols = int(np.exp(rng.uniform(np.log(8), np.log(256))))
        cases.append((rows, cols, KINDS[i % 3], EPS_GRID[i % 5], Q_GRID[(i // 5) % 5], i))
    return cases


def _sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def run_case(case):
    import ebcc
    rows, cols, kind, eps, q, seed = case
    a = fields.small_field(kind, rows, cols, seed)
    try:
        blob = ebcc.compress(a, rel_error=eps, q=q)
        err = None
    except ebcc.EbccError as exc:  # recorded, e.g. ResidualInsufficient
        blob, err = b"", type(exc).__name__
    return {"rows": rows, "cols": cols, "kind": kind, "eps": eps, "q": q, "seed": seed,
            "input_sha": _sha(np.ascontiguousarray(a).tobytes()),
            "container_sha": _sha(blob), "container_len": len(blob), "error": err}


def signed_zero_fields():
    out = []
    p = fields.precip_like(96, 160, seed=77)           # many +0.0 at the minimum
    idx = np.flatnonzero(p.reshape(-1) == 0)[:50]
    neg = p.copy().reshape(-1)
    neg[idx[::2]] = np.float32(-0.0)                   # mixed signed zeros at the minimum
    out.append(("precip_mixed_signed_zeros", neg.reshape(p.shape)))
    allneg = p.copy().reshape(-1)
    allneg[allneg == 0] = np.float32(-0.0)              # every zero negative
    out.append(("precip_all_negative_zeros", allneg.reshape(p.shape)))
    m = -fields.precip_like(64, 64, seed=78)            # zeros at the MAXIMUM (negated field)
    out.append(("negated_precip_zero_max", m.astype(np.float32)))
    return out


if __name__ == "__main__":
    ebcc = import_reference()
    cases = fuzz_cases()
    with mp.get_context("fork").Pool(len(os.sched_getaffinity(0))) as pool:
        res = pool.map(run_case, cases, chunksize=8)
    with open(os.path.join(HERE, "fuzz.json"), "w") as fh:
        json.dump(res, fh, indent=0)
    print(f"fuzz: {len(res)} cases, {sum(r['error'] is not None for r in res)} errors")
    edge = []
    for name, a in signed_zero_fields():
        blob = ebcc.compress(a, rel_error=0.01)
        mn = a.min()
        edge.append({"name": name, "rows": a.shape[0], "cols": a.shape[1],
                     "input_sha": _sha(np.ascontiguousarray(a).tobytes()), "eps": 0.01,
                     "reference_vmin_signbit": bool(np.signbit(mn)),
                     "container_sha": _sha(blob), "container_len": len(blob)})
    from ebcc.core import flatten_chunk
    from ebcc.pipeline import EbccParams, compress_chunk
    a = fields.temperature_like(721, 1440, seed=5, mean=250.0, std=10.0)
    cc = compress_chunk(flatten_chunk(a.reshape(1, 1, 721, 1440)),
                        EbccParams(epsilon_rel=0.01, r0=218576.84210526317))
    edge.append({"name": "floordiv_r0", "rows": 721, "cols": 1440,
                 "input_sha": _sha(np.ascontiguousarray(a).tobytes()), "eps": 0.01,
                 "r0": 218576.84210526317, "mode": int(cc.mode), "base_len": cc.base_len,
                 "resid_len": cc.residual_len, "payload_sha": _sha(cc.payload)})
    with open(os.path.join(HERE, "edge.json"), "w") as fh:
        json.dump(edge, fh, indent=1)
    print(json.dumps(edge, indent=1))
