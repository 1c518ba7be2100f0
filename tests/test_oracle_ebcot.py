"""CPU checks of the oracle's opt-in JPEG2000-style base layer (oracle/ebcot_oracle.c).

Parity is UNPINNED for this codec: the reference has no JPEG2000 base layer
(SPEC.md:261).  What can be checked without one are the algorithm's own
invariants: the MQ coder decodes what it encoded, the tier-1 coder's full
stream reconstructs every coefficient within one quantisation step, budgeted
streams are unit-aligned byte prefixes of the full stream whose error shrinks
as the budget grows, and the two-layer compressor built on it holds the
reference's error bound.
"""

import numpy as np
import pytest


@pytest.fixture(scope="module")
def o():
    from oracle import oracle
    oracle.build()
    return oracle


def test_mq_round_trip(o):
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = int(rng.integers(1, 4000))
        bits = (rng.random(n) < rng.uniform(0.01, 0.99)).astype(np.uint8)
        cx = rng.integers(0, 19, n).astype(np.uint8)
        assert np.array_equal(o.mq_decode(o.mq_encode(bits, cx), cx), bits)


def _pyramid(o, r, c, seed):
    from paper_2510_22265_b200 import fields
    a = fields.small_field("smooth", r, c, seed).astype(np.float64)
    norm = (a - a.min()) / (a.max() - a.min())
    lev = o.lib().eo_clamp_levels(r, c, o.default_levels(r, c))
    return o.forward_dwt(norm, lev)


@pytest.mark.parametrize("shape", [(24, 40), (64, 64), (100, 130), (17, 9), (2, 50), (96, 180)])
def test_tier1_full_stream_and_prefixes(o, shape):
    r, c = shape
    pyr, lev = _pyramid(o, r, c, 3)
    full = o.ebcot_encode(pyr, lev)
    step = 2.0 ** (np.floor(np.log2(np.abs(pyr).max())) - 23)
    assert np.abs(o.ebcot_decode(full, r, c) - pyr).max() <= step
    errs = []
    for b in (12, 40, 150, 600, 2500, 10000, len(full)):
        s = o.ebcot_encode(pyr, lev, b)
        assert len(s) <= max(b, 12)
        assert len(s) == 12 or full[: len(s)] == s
        errs.append(np.abs(o.ebcot_decode(s, r, c) - pyr).max())
    assert all(e2 <= e1 for e1, e2 in zip(errs, errs[1:]))


def test_blocks_tile_the_pyramid(o):
    for r, c in ((721, 1440), (33, 70), (5, 5)):
        lev = o.lib().eo_clamp_levels(r, c, o.default_levels(r, c))
        cover = np.zeros((r, c), np.int32)
        for r0, c0, h, w, _ in o.ebcot_blocks(r, c, lev):
            assert 0 < h <= 64 and 0 < w <= 64
            cover[r0:r0 + h, c0:c0 + w] += 1
        assert (cover == 1).all()


def test_two_layer_compress_holds_the_bound(o):
    import paper_2510_22265_b200 as ebcc
    from paper_2510_22265_b200 import fields
    for kind in ("smooth", "precip", "vortex"):
        for eps in (0.1, 0.01, 0.001):
            a = np.stack([fields.small_field(kind, 64, 96, s) for s in range(2)])
            blob = o.compress(a, rel_error=eps, base_codec="ebcot")
            assert blob[4:6] == b"\x02\x00"
            out = o.decompress(blob).reshape(a.shape)
            assert ebcc.error_stats(a, out).rel_max <= eps
