"""Pin the CPU oracle to the reference: every fixture in tests/golden/ was
produced by running the reference (tests/golden/make_golden.py); the oracle
must reproduce it bit for bit — coefficients, streams, probe order, containers.
"""

import hashlib

import numpy as np
import pytest

import golden_inputs as gi


def _bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


class TestDwt:
    def test_forward_and_inverse_bitwise(self, oracle, golden_dwt):
        meta = golden_dwt["meta"]
        for i, (r, c, levels, dflt) in enumerate(meta):
            x = gi.dwt_input(i)
            assert bytes.fromhex(gi.sha(x)) == golden_dwt[f"xsha{i}"].tobytes()
            assert oracle.default_levels(int(r), int(c)) == dflt
            coef, lv = oracle.forward_dwt(x)
            assert lv == levels
            assert _bits_equal(coef, golden_dwt[f"c{i}"]), f"forward {r}x{c}"
            y = oracle.inverse_dwt(golden_dwt[f"c{i}"], int(levels))
            assert _bits_equal(y, golden_dwt[f"y{i}"]), f"inverse {r}x{c}"

    def test_level_policy_kats(self, oracle):
        # test_dwt.py:127-137 style: depth = clamp(floor(log2 min) - 2, 1, 5)
        assert oracle.default_levels(8, 8) == 1
        assert oracle.default_levels(33, 17) == 2
        assert oracle.default_levels(721, 1440) == 5
        assert oracle.default_levels(1, 16) == 1
        assert oracle.default_levels(4096, 4096) == 5


class TestSpiht:
    def test_streams_bitwise(self, oracle, golden_spiht):
        meta = golden_spiht["meta"]
        for i, (r, c, seed, levels) in enumerate(meta):
            coef = golden_spiht[f"coef{i}"]
            x, lv = oracle.forward_dwt(gi.spiht_input(i))
            assert _bits_equal(x, coef)
            full = oracle.spiht_encode(coef, int(levels))
            assert full == golden_spiht[f"full{i}"].tobytes(), f"full stream case {i}"
            deep = oracle.spiht_encode(coef, int(levels), planes=32)
            assert deep == golden_spiht[f"deep{i}"].tobytes(), f"deep stream case {i}"
            for b in golden_spiht[f"budgets{i}"]:
                got = oracle.spiht_encode(coef, int(levels), max_bytes=int(b))
                assert got == golden_spiht[f"bud{i}_{int(b)}"].tobytes(), f"case {i} budget {b}"
                assert got == full[: len(got)], "budgeted stream is a byte prefix"

    def test_prefix_decodes_and_n_last(self, oracle, golden_spiht):
        meta = golden_spiht["meta"]
        for i, (r, c, seed, levels) in enumerate(meta):
            deep = golden_spiht[f"deep{i}"].tobytes()
            full = golden_spiht[f"full{i}"].tobytes()
            for cut, nl in golden_spiht[f"nlast{i}"]:
                cut, nl = int(cut), int(nl)
                if cut < 0:
                    dec, n_last = oracle.decode_with_plane(full, int(r), int(c))
                    ref = golden_spiht[f"decfull{i}"]
                else:
                    dec, n_last = oracle.decode_with_plane(deep, int(r), int(c), cut)
                    ref = golden_spiht[f"dec{i}_{cut}"]
                assert _bits_equal(dec, ref), f"case {i} cut {cut}"
                assert (-999 if n_last is None else n_last) == nl, f"n_last case {i} cut {cut}"

    def test_budget_for_ratio_kats(self, oracle):
        # test_base_codec.py:90-94 and CPython float floor-division corner cases
        assert oracle.budget_for_ratio(8, 8, 1.0) == 256
        assert oracle.budget_for_ratio(8, 8, 1000.0) == 12
        assert oracle.budget_for_ratio(8, 8, 0.99) == -1
        for ratio in (218576.84210526317, 3.7, 10.0, 1.0000001, 123456.789):
            raw = 721 * 1440 * 4
            assert oracle.budget_for_ratio(721, 1440, ratio) == max(12, int(raw // ratio))


def _check_case(oracle, case, arr):
    if "error" in case:
        with pytest.raises(Exception) as ei:
            oracle.compress(arr, case["eps"], case["q"], case.get("chunk_shape"))
        assert type(ei.value).__name__ == case["error"]
        return
    buf = oracle.compress(arr, case["eps"], case["q"], case.get("chunk_shape"))
    assert hashlib.sha256(buf).hexdigest() == case["container_sha"]
    if case.get("container"):
        assert buf.hex() == case["container"]
    out = oracle.decompress(buf)
    assert gi.sha(out) == case["decoded_sha"]


class TestChunks:
    def test_small_chunk_containers(self, oracle, golden_chunks):
        for case in golden_chunks["chunks"]:
            _check_case(oracle, case, gi.chunk_input(case))

    def test_probe_order_matches_reference(self, oracle, golden_chunks):
        """The feedback searches must visit the reference's budgets in the
        reference's order with identical q_achieved."""
        for case in golden_chunks["chunks"]:
            a = gi.chunk_input(case)
            if a.size < 1 or float(a.max()) - float(a.min()) < 1e-30:
                continue
            r = oracle.compress_chunk(a, case["eps"], case["q"], trace=True)
            assert [b for b, _ in r["base_trace"]] == [t[0] for t in case["base_trace"]]
            assert [q for _, q in r["base_trace"]] == [t[1] for t in case["base_trace"]]
            assert r["trunc_trace"] == case["trunc_trace"]

    def test_grids(self, oracle, golden_chunks):
        for case in golden_chunks["grids"]:
            arr = gi.grid_input(case["name"])
            assert gi.sha(arr) == case["input_sha"]
            _check_case(oracle, case, arr)


@pytest.mark.slow
def test_large_config_fields(oracle, golden_large):
    for case in golden_large[:1]:
        arr = gi.large_input(case["name"])
        assert gi.sha(arr) == case["input_sha"]
        r = oracle.compress_chunk(arr, case["eps"], case["q"], trace=True)
        assert [b for b, _ in r["base_trace"]] == [t[0] for t in case["base_trace"]]
        assert r["trunc_trace"] == case["trunc_trace"]
        _check_case(oracle, case, arr)
