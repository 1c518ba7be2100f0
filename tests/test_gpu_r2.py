"""GPU parity, round 2: the reference's own edge-case distribution, every field
of the BASELINE.json configurations, stress, stream and multi-process paths.

* fuzz.json / edge.json — made by the UNMODIFIED reference
  (tests/golden/make_golden_fuzz.py): the error-bound fuzz distribution of
  pkg/tests/test_acceptance.py:48-80 (1000 chunks, sizes 8..256, 3 kinds x
  5 eps x 5 q), signed zeros at the extrema, and a custom r0 whose first
  budget needs CPython float floor division (base_codec.py:38).
* oracle_configs.json — the C oracle (pinned to the reference's goldens) on
  every configs[1] level, configs[2] step, configs[3] variable and the first
  64 configs[4] sweep fields (tools/oracle_fixtures_r2.py).
"""

import hashlib
import json
import os

import numpy as np
import pytest

import golden_inputs as gi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")

pytestmark = pytest.mark.gpu


def _load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def _sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def _field_containers(stack, eps, q=1 - 1e-5, **kw):
    """One batched device call over `stack`; the single-field container of
    every chunk, as the reference's api.compress(field) would write it."""
    from paper_2510_22265_b200.chunk import EbccParams
    from paper_2510_22265_b200.container import RECORD_DTYPE, assemble
    from paper_2510_22265_b200.pipeline import compress_batch
    recs, offs, pay, st = compress_batch(np.ascontiguousarray(stack), EbccParams(eps, q, **kw))
    assert st == 0
    n, rows, cols = stack.shape
    dims = (1, 1, rows, cols)
    out = []
    for i in range(n):
        r = np.zeros(1, RECORD_DTYPE)
        for k in ("mode", "vmin", "vmax", "base_len", "resid_len"):
            r[k] = recs[i][k]
        r["eps"], r["q"] = eps, q
        out.append(assemble(dims, dims, r, pay, offs[i:i + 1]))
    return out


def test_acceptance_fuzz_distribution_vs_reference():
    """1000 fuzzed chunks (test_acceptance.py:48-80's distribution, this
    repo's generators): every container equals the reference's byte for
    byte, and every decoded point honours the bound."""
    import paper_2510_22265_b200 as ebcc
    from paper_2510_22265_b200 import fields
    bad = []
    worst = 0.0
    for c in _load("fuzz.json"):
        a = fields.small_field(c["kind"], c["rows"], c["cols"], c["seed"])
        assert gi.sha(a) == c["input_sha"]
        try:
            blob = ebcc.compress(a, rel_error=c["eps"], q=c["q"])
        except ebcc.EbccError as exc:
            if type(exc).__name__ != c["error"]:
                bad.append((c["seed"], "raised", type(exc).__name__))
            continue
        if c["error"] is not None or _sha(blob) != c["container_sha"]:
            bad.append((c["seed"], c["rows"], c["cols"], c["kind"], c["eps"], c["q"],
                        len(blob), c["container_len"]))
            continue
        st = ebcc.error_stats(a, ebcc.decompress(blob).reshape(a.shape))
        worst = max(worst, st.rel_max / c["eps"])
    assert not bad, f"{len(bad)} of 1000 differ: {bad[:6]}"
    assert worst <= 1.0


def test_edge_cases_vs_reference():
    """Signed zeros at the minimum / maximum and the floor-division corner."""
    import paper_2510_22265_b200 as ebcc
    from paper_2510_22265_b200 import fields
    from paper_2510_22265_b200.chunk import EbccParams
    from paper_2510_22265_b200.pipeline import compress_batch
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "mgf", os.path.join(GOLDEN, "make_golden_fuzz.py"))
    mgf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mgf)
    arrays = dict(mgf.signed_zero_fields())
    bad = []
    for c in _load("edge.json"):
        if c["name"] == "floordiv_r0":
            a = fields.temperature_like(721, 1440, seed=5, mean=250.0, std=10.0)
            assert gi.sha(a) == c["input_sha"]
            recs, offs, pay, st = compress_batch(a[None], EbccParams(0.01, r0=c["r0"]))
            r = recs[0]
            if (int(r["mode"]), int(r["base_len"]), int(r["resid_len"])) != \
                    (c["mode"], c["base_len"], c["resid_len"]) or _sha(bytes(pay)) != c["payload_sha"]:
                bad.append(("floordiv_r0", int(r["mode"]), int(r["base_len"]), c["base_len"]))
            continue
        a = arrays[c["name"]]
        assert gi.sha(a) == c["input_sha"]
        blob = ebcc.compress(a, rel_error=c["eps"])
        if _sha(blob) != c["container_sha"]:
            bad.append((c["name"], len(blob), c["container_len"]))
        out = ebcc.decompress(blob).reshape(a.shape)
        assert ebcc.error_stats(a, out).rel_max <= c["eps"]
    assert not bad, bad


@pytest.mark.parametrize("config", ["configs[1]", "configs[2]", "configs[3]", "configs[4]"])
def test_every_config_field_vs_oracle(config):
    """Every field of the configuration in ONE batched device call (lanes,
    multi-batch plans, incremental and abortable probes, candidate pruning):
    each field's container equals the oracle's single-field container."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "ofx", os.path.join(REPO, "tools", "oracle_fixtures_r2.py"))
    ofx = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ofx)
    cases = [c for c in _load("oracle_configs.json") if c["config"] == config]
    assert cases
    stack = np.stack([ofx.field_of((config, c["index"])) for c in cases])
    for a, c in zip(stack, cases):
        assert gi.sha(a) == c["input_sha"], (config, c["index"])
    got = _field_containers(stack, 0.01)
    bad = [(c["index"], len(b), c["container_len"]) for b, c in zip(got, cases)
           if _sha(b) != c["container_sha"]]
    assert not bad, f"{config}: {len(bad)} of {len(cases)} differ: {bad[:6]}"


def test_repeated_runs_are_identical():
    """50 x the 37-level batch: the same bytes every time (races in the
    cluster list machines or the device controller would show here)."""
    import paper_2510_22265_b200 as ebcc
    from paper_2510_22265_b200 import fields
    levels = fields.config2_levels()
    first = ebcc.compress(levels, 0.01)
    dec = ebcc.decompress(first).tobytes()
    for _ in range(49):
        blob = ebcc.compress(levels, 0.01)
        assert blob == first
    assert ebcc.decompress(first).tobytes() == dec


def test_default_stream_zero():
    """set_stream(0) (torch's default stream) works: the library keeps its
    own capturable stream and orders it after the caller's."""
    from paper_2510_22265_b200 import _lib, fields
    from paper_2510_22265_b200.chunk import EbccParams
    from paper_2510_22265_b200.pipeline import compress_batch
    stack = np.stack([fields.small_field("smooth", 64, 96, s) for s in range(3)])
    want = compress_batch(stack, EbccParams(0.01), _lib.Context(0))
    ctx = _lib.Context(0)
    ctx.set_stream(0)
    got = compress_batch(stack, EbccParams(0.01), ctx)
    assert bytes(got[2]) == bytes(want[2])
    assert np.array_equal(got[0]["base_len"], want[0]["base_len"])


def _dist_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)  # both ranks on the one GPU; collectives over gloo
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2510_22265_b200 import distributed, fields
    a = np.stack([fields.small_field(k, 72, 120, s) for s in range(3)
                  for k in ("smooth", "precip", "vortex")]).reshape(3, 3, 72, 120)
    blob = distributed.compress(a, rel_error=0.01)
    if rank == 0:
        with open(os.path.join(out_dir, "c.bin"), "wb") as fh:
            fh.write(blob)
    out = distributed.decompress(blob if rank == 0 else None)
    if rank == 0:
        np.save(os.path.join(out_dir, "d.npy"), out)
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_world2_equals_single_process(tmp_path):
    """The multi-GPU public API with world size 2 (both ranks on cuda:0,
    gloo collectives): the container and the decoded array equal the
    single-process GPU results."""
    import socket

    import torch.multiprocessing as mp

    import paper_2510_22265_b200 as ebcc
    from paper_2510_22265_b200 import fields
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(_dist_worker, args=(2, port, str(tmp_path)), nprocs=2,
                       start_method="spawn")
    a = np.stack([fields.small_field(k, 72, 120, s) for s in range(3)
                  for k in ("smooth", "precip", "vortex")]).reshape(3, 3, 72, 120)
    want = ebcc.compress(a, rel_error=0.01)
    got = open(tmp_path / "c.bin", "rb").read()
    assert got == want
    assert np.array_equal(np.load(tmp_path / "d.npy"), ebcc.decompress(want))
