"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden fixtures and against the CPU oracle.  Bit-exact throughout: float64
coefficients compared as bytes, streams and containers byte for byte.
"""

import hashlib
import os

import numpy as np
import pytest

import golden_inputs as gi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2510_22265_b200 import _lib
    return _lib.context(0)


@pytest.fixture(scope="module")
def ebcc():
    import paper_2510_22265_b200 as e
    return e


def _same(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def test_dwt_bitwise(ctx, golden_dwt):
    bad = []
    for i, (r, c, levels, dflt) in enumerate(golden_dwt["meta"]):
        x = gi.dwt_input(i)
        got = ctx.dwt(x, int(levels), inverse=False)[0]
        if not _same(got, golden_dwt[f"c{i}"]):
            bad.append(("fwd", int(r), int(c), float(np.abs(got - golden_dwt[f"c{i}"]).max())))
        y = ctx.dwt(golden_dwt[f"c{i}"], int(levels), inverse=True)[0]
        if not _same(y, golden_dwt[f"y{i}"]):
            bad.append(("inv", int(r), int(c), float(np.abs(y - golden_dwt[f"y{i}"]).max())))
    assert not bad, bad


def test_dwt_batched_matches_single(ctx):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((5, 37, 53)) * 100
    batch = ctx.dwt(x, 3, inverse=False)
    for k in range(5):
        assert _same(batch[k], ctx.dwt(x[k], 3, inverse=False)[0])


def test_spiht_streams_bitwise(ctx, golden_spiht):
    bad = []
    for i, (r, c, seed, levels) in enumerate(golden_spiht["meta"]):
        coef = golden_spiht[f"coef{i}"]
        full = ctx.spiht_encode(coef, int(levels), 24)
        if full != golden_spiht[f"full{i}"].tobytes():
            bad.append(("full", i, len(full), golden_spiht[f"full{i}"].size))
        deep = ctx.spiht_encode(coef, int(levels), 32)
        if deep != golden_spiht[f"deep{i}"].tobytes():
            bad.append(("deep", i, len(deep), golden_spiht[f"deep{i}"].size))
        for b in golden_spiht[f"budgets{i}"]:
            ref = golden_spiht[f"bud{i}_{int(b)}"].tobytes()
            if full[: len(ref)] != ref:
                bad.append(("budget", i, int(b)))
    assert not bad, bad


def test_spiht_prefix_decode_bitwise(ctx, golden_spiht):
    bad = []
    for i, (r, c, seed, levels) in enumerate(golden_spiht["meta"]):
        deep = golden_spiht[f"deep{i}"].tobytes()
        full = golden_spiht[f"full{i}"].tobytes()
        for cut, nl in golden_spiht[f"nlast{i}"]:
            cut, nl = int(cut), int(nl)
            if cut < 0:
                dec, n_last = ctx.spiht_decode(full, int(r), int(c))
                ref = golden_spiht[f"decfull{i}"]
            else:
                dec, n_last = ctx.spiht_decode(deep, int(r), int(c), cut)
                ref = golden_spiht[f"dec{i}_{cut}"]
            if not _same(dec, ref) or (-999 if n_last is None else n_last) != nl:
                bad.append((i, cut, n_last, nl, int((dec != ref).sum())))
    assert not bad, bad


def test_inverse_dwt_through_production_kernel(ctx, golden_spiht):
    """The inverse transform the product runs (idwt_fused.cuh level kernels,
    closed-form decode on load; dwt.py:202-216 / base_codec.py:70-84) on
    every golden stream prefix, lower-bound and midpoint dequantisation,
    bit-identical to the oracle's inverse_dwt of the reference's decoded
    coefficients (oracle inverse pinned by the dwt goldens)."""
    from oracle import oracle
    oracle.build()
    bad = []
    for i, (r, c, seed, levels) in enumerate(golden_spiht["meta"]):
        deep = golden_spiht[f"deep{i}"].tobytes()
        full = golden_spiht[f"full{i}"].tobytes()
        for cut, nl in golden_spiht[f"nlast{i}"]:
            cut, nl = int(cut), int(nl)
            if cut < 0:
                data, pre, coef = full, None, golden_spiht[f"decfull{i}"]
            else:
                data, pre, coef = deep, cut, golden_spiht[f"dec{i}_{cut}"]
            for mid in (False, True):
                cf = np.array(coef, np.float64)
                if mid and nl != -999:
                    cf = cf + np.sign(cf) * float(np.ldexp(0.5, nl))
                want = oracle.inverse_dwt(cf, int(levels))
                got = ctx.decode_field(data, int(r), int(c), pre, midpoint=mid)
                if not _same(got, want):
                    bad.append((i, cut, mid, int((got != want).sum())))
    assert not bad, bad


def _run_case(ebcc, case, arr):
    """Returns None on parity, else a description of the first difference."""
    kw = dict(rel_error=case["eps"], q=case["q"], chunk_shape=case.get("chunk_shape"))
    if "error" in case:
        try:
            ebcc.compress(arr, **kw)
        except ebcc.EbccError as exc:
            return None if type(exc).__name__ == case["error"] else f"raised {exc!r}"
        return f"expected {case['error']}"
    try:
        buf = ebcc.compress(arr, **kw)
    except ebcc.EbccError as exc:
        return f"raised {exc!r}"
    if hashlib.sha256(buf).hexdigest() != case["container_sha"]:
        from paper_2510_22265_b200.container import read_file
        chunks, _, _ = read_file(buf)
        return ("container", [int(c.mode) for c in chunks], [c.base_len for c in chunks],
                [c.residual_len for c in chunks], case["modes"], case["base_lens"],
                case["resid_lens"])
    out = ebcc.decompress(buf)
    if gi.sha(out) != case["decoded_sha"]:
        return "decoded"
    return None


def test_small_chunk_containers(ebcc, golden_chunks):
    bad = []
    for case in golden_chunks["chunks"]:
        r = _run_case(ebcc, case, gi.chunk_input(case))
        if r is not None:
            bad.append((case["kind"], case["rows"], case["cols"], case["eps"], case["q"], r))
    assert not bad, f"{len(bad)} mismatches: {bad[:8]}"


def test_probe_counts_match_reference(golden_chunks):
    """P_base / P_trunc per chunk equal the reference's probe traces."""
    from paper_2510_22265_b200 import fields  # noqa: F401
    from paper_2510_22265_b200.chunk import EbccParams
    from paper_2510_22265_b200.pipeline import compress_batch
    bad = []
    for case in golden_chunks["chunks"]:
        if "error" in case or case["kind"] == "const":
            continue
        a = gi.chunk_input(case)
        recs, _, _, st = compress_batch(a[None], EbccParams(case["eps"], case["q"]),
                                        full_search=True)
        if st != 0:
            continue
        nb, nt = int(recs[0]["n_base_probes"]), int(recs[0]["n_trunc_probes"])
        if nb != len(case["base_trace"]) or nt != len(case["trunc_trace"]):
            bad.append((case["rows"], case["cols"], nb, len(case["base_trace"]), nt,
                        len(case["trunc_trace"])))
    assert not bad, bad


def test_grids(ebcc, golden_chunks):
    bad = []
    for case in golden_chunks["grids"]:
        arr = gi.grid_input(case["name"])
        assert gi.sha(arr) == case["input_sha"]
        r = _run_case(ebcc, case, arr)
        if r is not None:
            bad.append((case["name"], r))
    assert not bad, bad


def test_batched_equals_single(ebcc):
    """One batch of many chunks gives the same bytes as one call per chunk."""
    from paper_2510_22265_b200 import fields
    # 20 chunks: large enough for the concurrent two-lane split
    stack = np.stack([fields.small_field(k, 40, 56, s) for s, k in
                      enumerate(["smooth", "spiky", "precip", "noise"] * 5)])
    whole = ebcc.compress(stack, 0.01)
    parts = [ebcc.compress(stack[i], 0.01) for i in range(len(stack))]
    from paper_2510_22265_b200.container import read_file
    chunks, _, _ = read_file(whole)
    for i, blob in enumerate(parts):
        c1, _, _ = read_file(blob)
        assert c1[0].payload == chunks[i].payload


@pytest.mark.parametrize("eps", [0.001, 0.01, 0.1])
def test_candidate_pruning_keeps_bytes(ebcc, eps):
    """Stopping a search whose candidate can no longer win (the default)
    gives the same records and payload as running every probe of the
    reference's searches (EBCC_FULL_SEARCH), with no more probes."""
    from paper_2510_22265_b200 import fields
    from paper_2510_22265_b200.chunk import EbccParams
    from paper_2510_22265_b200.pipeline import compress_batch
    stack = np.stack([fields.small_field(k, 96, 160, 100 + s) for s, k in
                      enumerate(["smooth", "spiky", "precip", "noise"] * 5)])
    stack = np.concatenate([stack, fields.temperature_like(96, 160, seed=7)[None],
                            fields.precip_like(96, 160, seed=8)[None]])
    p = EbccParams(eps)
    r_fast, o_fast, pay_fast, st_fast = compress_batch(stack, p)
    r_full, o_full, pay_full, st_full = compress_batch(stack, p, full_search=True)
    assert st_fast == st_full
    for key in ("mode", "base_len", "resid_len", "status"):
        assert np.array_equal(r_fast[key], r_full[key]), key
    assert np.array_equal(o_fast, o_full)
    assert bytes(pay_fast) == bytes(pay_full)
    assert np.all(r_fast["n_base_probes"] <= r_full["n_base_probes"])
    assert np.all(r_fast["n_trunc_probes"] <= r_full["n_trunc_probes"])


def test_full_size_other_eps_vs_oracle_fixtures(ebcc):
    """configs[1] levels at eps 0.1% and 10% (BASELINE.json's other targets):
    containers equal the C oracle's (tests/golden/oracle_eps.json, made by
    tools/oracle_fixture_eps.py), alone and inside one batched call of all
    37 levels (incremental probes, candidate pruning and abortable probes
    across many chunks and both lanes)."""
    import hashlib
    import json
    import os
    from paper_2510_22265_b200 import fields
    from paper_2510_22265_b200.container import read_file
    with open(os.path.join(os.path.dirname(__file__), "golden", "oracle_eps.json")) as fh:
        cases = json.load(fh)
    levels = fields.config2_levels()[0]
    bad = []
    for eps in sorted({c["eps"] for c in cases}):
        whole, _, _ = read_file(ebcc.compress(levels[None], rel_error=eps))
        for case in (c for c in cases if c["eps"] == eps):
            a = levels[case["level"]]
            assert gi.sha(a) == case["input_sha"], case["name"]
            blob = ebcc.compress(a, rel_error=eps)
            if hashlib.sha256(blob).hexdigest() != case["container_sha"]:
                bad.append((case["name"], eps, "single", len(blob), case["container_len"]))
            single, _, _ = read_file(blob)
            if whole[case["level"]].payload != single[0].payload:
                bad.append((case["name"], eps, "batched"))
    assert not bad, bad


def test_large_golden(ebcc, golden_large):
    bad = []
    for case in golden_large:
        arr = gi.large_input(case["name"])
        assert gi.sha(arr) == case["input_sha"]
        r = _run_case(ebcc, case, arr)
        if r is not None:
            bad.append((case["name"], r))
    assert not bad, bad


def test_full_size_config3_config4_vs_oracle_fixtures(ebcc):
    """Largest BASELINE.json shapes (configs[3]: 2881x5760; configs[2] steps):
    container bytes equal the C oracle's (tests/golden/oracle_large.json,
    made by tools/oracle_fixture_c4.py; the oracle is pinned to the
    reference's own goldens)."""
    import hashlib
    import json
    import os
    from paper_2510_22265_b200 import fields
    with open(os.path.join(os.path.dirname(__file__), "golden", "oracle_large.json")) as fh:
        cases = json.load(fh)
    bad = []
    big = {}
    for case in cases:
        name = case["name"]
        if name.startswith("config4_var"):
            arr = fields.config4_field(int(name[len("config4_var"):]))
        else:
            t = int(name[len("config3_step"):])
            arr = fields.precip_like(fields.GRID_025[0], fields.GRID_025[1], seed=2000 + t)
        assert gi.sha(arr) == case["input_sha"], name
        blob = ebcc.compress(arr, case["eps"], case["q"])
        if hashlib.sha256(blob).hexdigest() != case["container_sha"]:
            bad.append((name, len(blob), case["container_len"]))
        if name.startswith("config4_var"):
            big[name] = (arr, blob)
    assert not bad, bad
    # the configs[3] chunks in one call: several concurrent lanes and 7-CTA
    # list-machine clusters; every chunk's payload equals its single-call one
    from paper_2510_22265_b200.container import read_file
    names = sorted(big)
    whole, _, _ = read_file(ebcc.compress(np.stack([big[k][0] for k in names])))
    for i, k in enumerate(names):
        single, _, _ = read_file(big[k][1])
        assert whole[i].payload == single[0].payload, k


def test_random_fields_vs_oracle(ebcc, oracle):
    """Fresh random shapes/kinds/targets (not in the goldens): GPU container
    bytes equal the oracle's."""
    from paper_2510_22265_b200 import fields
    rng = np.random.default_rng(77)
    bad = []
    for i in range(40):
        r = int(rng.integers(3, 140))
        c = int(rng.integers(3, 140))
        kind = ["smooth", "spiky", "precip", "noise"][i % 4]
        eps = float(10 ** rng.uniform(-4, -0.5))
        q = float([1 - 1e-5, 1.0, 0.999, 0.9][i % 4])
        a = fields.small_field(kind, r, c, 9000 + i)
        try:
            want = oracle.compress(a, eps, q)
        except Exception as exc:
            want = type(exc).__name__
        try:
            got = ebcc.compress(a, eps, q)
        except ebcc.EbccError as exc:
            got = type(exc).__name__
        if got != want:
            bad.append((kind, r, c, eps, q))
    assert not bad, bad


def test_fma_corrected_division_is_exact(ctx):
    """The kernels replace x/SCALE and x/range by an FMA-corrected reciprocal
    multiply; it must equal IEEE division bit for bit (2^28 cases x 3)."""
    assert ctx.selftest_div(1 << 28, seed=20251020) == 0


def test_ingest_errors_from_device(ebcc):
    """Non-finite input is reported by the device ingest kernel with the
    reference's IngestError(index) (core.py:74-79), before param validation."""
    a = np.random.default_rng(1).standard_normal((3, 40, 50)).astype(np.float32)
    a[1, 7, 9] = np.nan
    a[2, 0, 0] = np.inf
    with pytest.raises(ebcc.IngestError) as ei:
        ebcc.compress(a, 0.01)
    assert ei.value.index == (1, 7, 9)
    with pytest.raises(ebcc.IngestError):
        ebcc.compress(a, 2.0)  # bad param too: ingest error wins, like the reference
    b = np.ones((20, 30), np.float32)
    b[-1, -1] = -np.inf
    with pytest.raises(ebcc.IngestError) as ei:
        ebcc.compress(b)
    assert ei.value.index == (19, 29)


@pytest.mark.gpu
def test_multi_batch_path_equals_single_batch(tmp_path):
    """Chunks split over several device batches (EBCC_MAX_BATCH, as when HBM
    bounds the batch) give the same container and decoded array."""
    import subprocess
    import sys
    script = r'''
import hashlib, sys
import numpy as np
sys.path.insert(0, "%s")
import paper_2510_22265_b200 as ebcc
from paper_2510_22265_b200 import fields
a = np.stack([fields.small_field(k, 48, 80, s) for s in range(3)
              for k in ("smooth", "precip", "noise")])[None]
blob = ebcc.compress(a, 0.01)
out = ebcc.decompress(blob)
print(hashlib.sha256(blob).hexdigest(), hashlib.sha256(out.tobytes()).hexdigest())
''' % REPO
    res = {}
    for mb in ("4096", "2"):
        env = dict(os.environ, EBCC_MAX_BATCH=mb)
        r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[mb] = r.stdout.split()
    assert res["4096"] == res["2"]
