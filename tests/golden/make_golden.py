"""Generate the golden fixtures under tests/golden/ by running the reference.

Run in the build container only (the reference lives at /root/reference and
does not travel to the GPU box):

    python tests/golden/make_golden.py            # small + medium fixtures
    python tests/golden/make_golden.py --large    # also the 721x1440 fields

The reference package is copied to a scratch directory and imported from
there (``/root/reference`` is read-only).  Inputs are produced by this repo's
own seeded generators (paper_2510_22265_b200/fields.py) and identified in the
fixtures by a SHA-256 of their float32 bytes, so a test can regenerate them and
prove it fed the same values.  What is stored per case:

* dwt.npz       forward coefficients and inverse outputs (float64 bytes)
* spiht.npz     full / deep / budgeted streams and prefix decodes (+ n_last)
* chunks.json   per-chunk containers (hex), decoded float32 SHA-256, and the
                feedback-probe trace: the ordered base budgets with their
                q_achieved and the ordered residual truncation offsets
* large.json    the same for the full-size fields (with --large)
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from paper_2510_22265_b200 import fields  # noqa: E402

SCRATCH = "/tmp/ebcc_ref_golden"


def import_reference():
    if not os.path.isdir(os.path.join(SCRATCH, "src", "ebcc")):
        shutil.rmtree(SCRATCH, ignore_errors=True)
        shutil.copytree("/root/reference/pkg", SCRATCH)
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    import ebcc  # noqa: F401
    return ebcc


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


DWT_SHAPES = [(2, 2), (7, 5), (8, 8), (33, 17), (1, 16), (16, 1), (45, 23),
              (45, 90), (3, 64), (64, 3), (1, 1), (2, 9), (5, 1), (1, 2),
              (17, 33), (64, 64), (13, 200)]


def make_dwt(ebcc):
    from ebcc.dwt import default_levels, forward_dwt, inverse_dwt
    out = {}
    meta = []
    for i, (r, c) in enumerate(DWT_SHAPES):
        x = np.random.default_rng(100 + i).standard_normal((r, c)) * 10.0
        pyr = forward_dwt(x)
        y = inverse_dwt(pyr)
        out[f"xsha{i}"] = np.frombuffer(bytes.fromhex(sha(x)), np.uint8)
        out[f"c{i}"] = pyr.coeffs
        out[f"y{i}"] = y
        meta.append((r, c, pyr.levels, default_levels(r, c)))
    out["meta"] = np.array(meta, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "dwt.npz"), **out)


SPIHT_CASES = [(8, 8, 0), (16, 16, 1), (33, 17, 2), (12, 20, 3), (1, 16, 4),
               (16, 1, 5), (22, 16, 6), (45, 23, 7), (5, 3, 8), (64, 48, 9),
               (2, 2, 10), (9, 30, 11)]


def make_spiht(ebcc):
    from ebcc import spiht
    from ebcc.dwt import forward_dwt
    out = {}
    meta = []
    for i, (r, c, seed) in enumerate(SPIHT_CASES):
        gen = np.random.default_rng(500 + seed)
        x = gen.standard_normal((r, c)) * (10.0 ** gen.uniform(-3, 3))
        pyr = forward_dwt(x)
        full = spiht.spiht_encode(pyr).data
        deep = spiht.spiht_encode(pyr, planes=spiht.DEEP_PLANES).data
        out[f"coef{i}"] = pyr.coeffs
        out[f"full{i}"] = np.frombuffer(full, np.uint8)
        out[f"deep{i}"] = np.frombuffer(deep, np.uint8)
        budgets = sorted({12, 13, 15, 20, 40, len(full) // 2, len(full) + 5})
        for b in budgets:
            out[f"bud{i}_{b}"] = np.frombuffer(spiht.spiht_encode(pyr, max_bytes=b).data, np.uint8)
        cuts = sorted({12, 13, 14, 17, len(deep) // 3, len(deep) // 2, len(deep) - 1, len(deep)})
        nl = []
        for cut in cuts:
            dec, n_last = spiht.decode_with_plane(deep, cut)
            out[f"dec{i}_{cut}"] = dec.coeffs
            nl.append((cut, -999 if n_last is None else n_last))
        # the 24-plane stream decoded whole: exercises zero-padded phantom planes
        dec, n_last = spiht.decode_with_plane(full)
        out[f"decfull{i}"] = dec.coeffs
        nl.append((-1, -999 if n_last is None else n_last))
        out[f"nlast{i}"] = np.array(nl, dtype=np.int64)
        out[f"budgets{i}"] = np.array(budgets, dtype=np.int64)
        meta.append((r, c, seed, pyr.levels))
    out["meta"] = np.array(meta, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "spiht.npz"), **out)


class Tracer:
    """Wraps the reference's probe functions to record the search order."""

    def __init__(self, ebcc):
        import ebcc.pipeline as pl
        self.pl = pl
        self.base_calls = []
        self.trunc_calls = []
        self._orig_base = pl.base_encode_budget
        self._orig_two = pl._reconstruct_two_layer

        def base(values, budget, epsilon):
            enc = self._orig_base(values, budget, epsilon)
            self.base_calls.append([int(budget), float(enc.q_achieved), len(enc.data)])
            return enc

        def two(stream_data, prefix_payload, base_field):
            self.trunc_calls.append(int(prefix_payload))
            return self._orig_two(stream_data, prefix_payload, base_field)

        pl.base_encode_budget = base
        pl._reconstruct_two_layer = two

    def reset(self):
        self.base_calls = []
        self.trunc_calls = []


def run_case(ebcc, tracer, arr, eps, q, chunk_shape=None):
    tracer.reset()
    t0 = time.perf_counter()
    try:
        buf = ebcc.compress(arr, rel_error=eps, q=q, chunk_shape=chunk_shape)
    except ebcc.EbccError as exc:
        return {"eps": eps, "q": q, "chunk_shape": chunk_shape,
                "input_sha": sha(arr), "shape": list(arr.shape),
                "error": type(exc).__name__, "message": str(exc),
                "base_trace": tracer.base_calls, "trunc_trace": tracer.trunc_calls}
    tc = time.perf_counter() - t0
    t0 = time.perf_counter()
    out = ebcc.decompress(buf)
    td = time.perf_counter() - t0
    from ebcc.container import read_file
    chunks, _, _ = read_file(buf)
    return {
        "eps": eps, "q": q, "chunk_shape": chunk_shape,
        "input_sha": sha(arr), "shape": list(arr.shape),
        "container": buf.hex() if len(buf) < 200000 else None,
        "container_sha": hashlib.sha256(buf).hexdigest(),
        "container_len": len(buf),
        "modes": [int(c.mode) for c in chunks],
        "base_lens": [int(c.base_len) for c in chunks],
        "resid_lens": [int(c.residual_len) for c in chunks],
        "decoded_sha": sha(out),
        "base_trace": tracer.base_calls,
        "trunc_trace": tracer.trunc_calls,
        "t_compress": tc, "t_decompress": td,
    }


def small_cases():
    cases = []
    shapes = [(8, 8), (16, 16), (24, 24), (32, 32), (40, 36), (33, 17), (17, 33),
              (48, 48), (64, 64), (13, 57), (100, 30), (1, 32), (32, 1), (2, 2),
              (3, 3), (4, 7), (1, 1), (1, 7), (9, 1), (5, 130), (96, 97), (16, 22),
              (128, 96), (11, 11)]
    kinds = ["smooth", "spiky", "precip", "noise"]
    epss = [0.001, 0.01, 0.1, 0.05, 0.005]
    qs = [1 - 1e-5, 1.0, 1 - 1e-3, 1 - 1e-7]
    k = 0
    for si, (r, c) in enumerate(shapes):
        for j in range(3):
            kind = kinds[(si + j) % 4]
            eps = epss[(si * 3 + j) % 5]
            q = qs[(si + 2 * j) % 4]
            cases.append(dict(kind=kind, rows=r, cols=c, seed=k, eps=eps, q=q))
            k += 1
    # constant and near-constant chunks
    cases.append(dict(kind="const", rows=12, cols=12, seed=0, eps=0.01, q=1 - 1e-5))
    # low q forces quantile violations -> TWO_LAYER with real truncation
    # searches; tiny epsilons push the residual to its 32-plane retry or to
    # ResidualInsufficient
    extra = [("spiky", 64, 64, 0.01, 0.99), ("noise", 50, 50, 0.05, 0.9),
             ("precip", 80, 120, 0.01, 0.999), ("smooth", 30, 30, 0.001, 0.5),
             ("noise", 20, 20, 1e-6, 0.5), ("smooth", 16, 16, 1e-8, 0.9),
             ("smooth", 8, 8, 1e-9, 1.0), ("spiky", 70, 45, 0.002, 0.95),
             ("noise", 33, 65, 0.02, 0.8), ("smooth", 24, 40, 1e-7, 0.99),
             ("precip", 64, 64, 0.05, 0.9), ("spiky", 128, 128, 0.01, 0.9999),
             ("noise", 12, 12, 1e-5, 0.7), ("smooth", 19, 23, 3e-7, 0.6)]
    for kind, r, c, eps, q in extra:
        cases.append(dict(kind=kind, rows=r, cols=c, seed=k, eps=eps, q=q))
        k += 1
    # intermittent fields at tiny epsilon: the 24-plane residual misses the
    # bound and the 32-plane retry runs (or nothing reaches it)
    retry = [(6, 4, 10031, 2.885257848246616e-09, 0.2629040297325119),
             (4, 8, 10271, 4.964730095971289e-10, 0.5109448128922991),
             (6, 20, 11187, 1.4107571980791546e-10, 0.31473287365529096),
             (5, 17, 11559, 1.6519739980192603e-10, 0.23800578479129655),
             (10, 21, 12099, 1.3438158903802087e-09, 0.20498950826866694),
             (11, 22, 12867, 6.865343887389856e-08, 0.22871610607679857)]
    for r, c, seed, eps, q in retry:
        cases.append(dict(kind="precip", rows=r, cols=c, seed=seed, eps=eps, q=q))
    return cases


def make_input(case):
    if case["kind"] == "const":
        return np.full((case["rows"], case["cols"]), 4.5, np.float32)
    return fields.small_field(case["kind"], case["rows"], case["cols"], case["seed"])


def grid_cases():
    """Multi-chunk grids with edge chunks (chunk_shape that does not divide)."""
    g1 = (np.random.default_rng(5).standard_normal((2, 2, 12, 12))).astype(np.float32)
    g2 = (np.random.default_rng(6).standard_normal((1, 2, 20, 16)) * 50 + 300).astype(np.float32)
    g3 = fields.small_field("smooth", 50, 70, 77).reshape(1, 1, 50, 70) * 10 + 5
    return [
        dict(name="g1", seed=5, eps=0.02, q=1 - 1e-5, chunk_shape=(1, 1, 6, 12), arr=g1),
        dict(name="g2", seed=6, eps=0.01, q=1 - 1e-5, chunk_shape=(1, 1, 10, 16), arr=g2),
        dict(name="g3", seed=77, eps=0.01, q=1 - 1e-5, chunk_shape=(1, 1, 16, 32), arr=g3),
        dict(name="g4", seed=6, eps=0.05, q=1 - 1e-5, chunk_shape=(1, 2, 7, 16), arr=g2),
    ]


def make_chunks(ebcc):
    tracer = Tracer(ebcc)
    res = []
    for case in small_cases():
        arr = make_input(case)
        r = run_case(ebcc, tracer, arr, case["eps"], case["q"])
        r.update({k: case[k] for k in ("kind", "rows", "cols", "seed")})
        res.append(r)
    for case in [dict(kind="smooth", rows=96, cols=192, seed=901, eps=0.01, q=1 - 1e-5),
                 dict(kind="precip", rows=181, cols=360, seed=902, eps=0.01, q=1 - 1e-5),
                 dict(kind="spiky", rows=120, cols=200, seed=903, eps=0.001, q=1 - 1e-5),
                 dict(kind="smooth", rows=181, cols=360, seed=904, eps=0.1, q=1 - 1e-5)]:
        arr = make_input(case)
        r = run_case(ebcc, tracer, arr, case["eps"], case["q"])
        r.update({k: case[k] for k in ("kind", "rows", "cols", "seed")})
        res.append(r)
    grids = []
    for g in grid_cases():
        r = run_case(ebcc, tracer, g["arr"], g["eps"], g["q"], g["chunk_shape"])
        r["name"] = g["name"]
        grids.append(r)
    with open(os.path.join(HERE, "chunks.json"), "w") as fh:
        json.dump({"chunks": res, "grids": grids}, fh)


def make_large(ebcc):
    tracer = Tracer(ebcc)
    res = []
    c1 = fields.config1_field()
    r = run_case(ebcc, tracer, c1, 0.01, 1 - 1e-5)
    r["name"] = "config1_721x1440_eps1pct"
    res.append(r)
    print("config1", r["t_compress"], r["container_len"], file=sys.stderr)
    lv = fields.config2_levels(levels=37)
    for lev, eps in ((0, 0.001), (18, 0.01), (36, 0.1)):
        a = lv[0, lev]
        r = run_case(ebcc, tracer, a, eps, 1 - 1e-5)
        r["name"] = f"config2_level{lev}_eps{eps}"
        res.append(r)
        print(r["name"], r["t_compress"], r["container_len"], file=sys.stderr)
    pr = fields.precip_like(721, 1440, seed=2000)
    r = run_case(ebcc, tracer, pr, 0.01, 1 - 1e-5)
    r["name"] = "config3_step0_eps1pct"
    res.append(r)
    with open(os.path.join(HERE, "large.json"), "w") as fh:
        json.dump(res, fh)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    ebcc = import_reference()
    todo = args.only.split(",") if args.only else ["dwt", "spiht", "chunks"]
    if "dwt" in todo:
        make_dwt(ebcc)
    if "spiht" in todo:
        make_spiht(ebcc)
    if "chunks" in todo:
        make_chunks(ebcc)
    if args.large or "large" in todo:
        make_large(ebcc)


if __name__ == "__main__":
    main()
