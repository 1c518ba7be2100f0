"""GPU checks of the opt-in JPEG2000-style base layer (base_codec="ebcot").

PARITY IS UNPINNED for this codec: the reference has no JPEG2000 base layer
(the paper used OpenJPEG).  The GPU codec is checked byte for
byte against the CPU oracle's independent restatement (oracle/ebcot_oracle.c,
itself checked for the algorithm's invariants in test_oracle_ebcot.py):
containers (search decisions from the GPU's closed-form prefix decode, the
oracle's from MQ decoding), decoded arrays (GPU MQ decoder), and the error
bound at every point.
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


@pytest.fixture(scope="module")
def oracle():
    from oracle import oracle as o
    o.build()
    return o


@pytest.mark.parametrize("kind", ["smooth", "precip", "vortex"])
@pytest.mark.parametrize("eps", [0.1, 0.01, 0.001])
def test_small_fields_vs_oracle(oracle, kind, eps):
    import paper_2510_22265_b200 as ebcc
    from paper_2510_22265_b200 import fields
    a = np.stack([fields.small_field(kind, 72, 120, s) for s in range(3)]).reshape(1, 3, 72, 120)
    got = ebcc.compress(a, rel_error=eps, base_codec="ebcot")
    want = oracle.compress(a, rel_error=eps, base_codec="ebcot")
    assert got[4:6] == b"\x02\x00"
    assert got == want
    out = ebcc.decompress(got)
    assert np.array_equal(out, oracle.decompress(want))
    assert ebcc.error_stats(a, out).rel_max <= eps


def test_edge_shapes_and_custom_chunks_vs_oracle(oracle):
    import paper_2510_22265_b200 as ebcc
    from paper_2510_22265_b200 import fields
    for r, c in ((1, 37), (5, 3), (17, 130), (65, 64), (130, 66)):
        a = fields.small_field("smooth", r, c, 7)
        got = ebcc.compress(a, rel_error=0.01, base_codec="ebcot")
        assert got == oracle.compress(a, rel_error=0.01, base_codec="ebcot"), (r, c)
        assert np.array_equal(ebcc.decompress(got), oracle.decompress(got))
    a = np.stack([fields.small_field("precip", 60, 90, s) for s in range(4)]).reshape(2, 2, 60, 90)
    got = ebcc.compress(a, rel_error=0.01, chunk_shape=(1, 2, 40, 50), base_codec="ebcot")
    want = oracle.compress(a, rel_error=0.01, chunk_shape=(1, 2, 40, 50), base_codec="ebcot")
    assert got == want
    assert np.array_equal(ebcc.decompress(got), oracle.decompress(want))


def test_full_size_fields_vs_oracle_fixtures():
    import importlib.util
    import paper_2510_22265_b200 as ebcc
    spec = importlib.util.spec_from_file_location(
        "ofe", os.path.join(REPO, "tools", "oracle_fixtures_ebcot.py"))
    ofe = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ofe)
    with open(os.path.join(GOLDEN, "oracle_ebcot.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        a = ofe.field_of(c["kind"], c["kw"])
        assert gi.sha(a) == c["input_sha"]
        blob = ebcc.compress(a, rel_error=c["eps"], base_codec="ebcot")
        assert hashlib.sha256(blob).hexdigest() == c["container_sha"], (c["kind"], len(blob),
                                                                      c["container_len"])
        out = ebcc.decompress(blob)
        assert gi.sha(out) == c["decoded_sha"]
        assert ebcc.error_stats(a, out.reshape(a.shape)).rel_max <= c["eps"]


def test_batched_stack_bound_and_ratio():
    """37 levels through one batched call: the bound at every point; the
    J2 base layer compresses at least as well as the reference's SPIHT base
    on these smooth fields (the paper's reason for a JPEG2000 base layer)."""
    import paper_2510_22265_b200 as ebcc
    from paper_2510_22265_b200 import fields
    levels = fields.config2_levels()
    blob = ebcc.compress(levels, rel_error=0.01, base_codec="ebcot")
    out = ebcc.decompress(blob).reshape(levels.shape)
    for k in range(levels.shape[0]):
        assert ebcc.error_stats(levels[k], out[k]).rel_max <= 0.01
    assert len(blob) < len(ebcc.compress(levels, rel_error=0.01))
