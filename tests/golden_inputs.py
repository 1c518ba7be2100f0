"""Regenerate the inputs the golden fixtures were made from (and prove it).

tests/golden/make_golden.py stores a SHA-256 of every float32 input it fed
the reference; these helpers rebuild the arrays with the repo's seeded
generators and assert the hash matches before any comparison is trusted.
"""

from __future__ import annotations

import hashlib

import numpy as np

from paper_2510_22265_b200 import fields

DWT_SHAPES = [(2, 2), (7, 5), (8, 8), (33, 17), (1, 16), (16, 1), (45, 23),
              (45, 90), (3, 64), (64, 3), (1, 1), (2, 9), (5, 1), (1, 2),
              (17, 33), (64, 64), (13, 200)]

SPIHT_CASES = [(8, 8, 0), (16, 16, 1), (33, 17, 2), (12, 20, 3), (1, 16, 4),
               (16, 1, 5), (22, 16, 6), (45, 23, 7), (5, 3, 8), (64, 48, 9),
               (2, 2, 10), (9, 30, 11)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dwt_input(i: int) -> np.ndarray:
    r, c = DWT_SHAPES[i]
    return np.random.default_rng(100 + i).standard_normal((r, c)) * 10.0


def spiht_input(i: int) -> np.ndarray:
    r, c, seed = SPIHT_CASES[i]
    gen = np.random.default_rng(500 + seed)
    return gen.standard_normal((r, c)) * (10.0 ** gen.uniform(-3, 3))


def chunk_input(case: dict) -> np.ndarray:
    if case["kind"] == "const":
        a = np.full((case["rows"], case["cols"]), 4.5, np.float32)
    else:
        a = fields.small_field(case["kind"], case["rows"], case["cols"], case["seed"])
    assert sha(a) == case["input_sha"], "regenerated input differs from the golden's"
    return a


def grid_input(name: str) -> np.ndarray:
    if name == "g1":
        return np.random.default_rng(5).standard_normal((2, 2, 12, 12)).astype(np.float32)
    if name in ("g2", "g4"):
        return (np.random.default_rng(6).standard_normal((1, 2, 20, 16)) * 50
                + 300).astype(np.float32)
    if name == "g3":
        return fields.small_field("smooth", 50, 70, 77).reshape(1, 1, 50, 70) * 10 + 5
    raise KeyError(name)


def large_input(name: str) -> np.ndarray:
    if name.startswith("config1"):
        return fields.config1_field()
    if name.startswith("config2_level"):
        lev = int(name.split("level")[1].split("_")[0])
        frac = lev / 36
        return fields.temperature_like(721, 1440, seed=1000 + lev, mean=200.0 + 100.0 * frac,
                                       std=2.0 + 18.0 * frac)
    if name.startswith("config3"):
        return fields.precip_like(721, 1440, seed=2000)
    raise KeyError(name)
