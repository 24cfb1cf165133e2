"""Pin the CPU oracle to the reference: replay every golden fixture (generated
by the unmodified reference, tests/golden/make_golden.py) through the numpy
restatement and the correctly rounded C restatement."""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import exact, polar_oracle as po
from tests.helpers import case, case_names, compare_codes


def test_fixture_host_recorded(golden):
    assert golden["__cpu_features__"].size > 0
    assert str(golden["__numpy__"])


@pytest.mark.parametrize("idx", range(12))
def test_numpy_oracle_encoder_matches_reference(golden, same_host_features, idx):
    c = case(golden, f"enc{idx}")
    T, d, m, n, lay = (int(v) for v in c["cfg"])
    s16 = po.scales_fp16(c["keys"], n, lay)
    assert np.array_equal(s16.view(np.uint16), c["scales"])
    a, r, clamped = po.encode_block(c["keys"], s16, m, n, lay)
    compare_codes(c["keys"], lay, m, n, s16, a, r, c["angle"], c["radius"], exact=same_host_features)
    if same_host_features:
        assert po.pack(a, m) == c["angle_stream"].tobytes()
        assert po.pack(r, n) == c["radius_stream"].tobytes()
    assert clamped == int(c["clamped"])
    assert np.array_equal(po.unpack(c["angle_stream"].tobytes(), m, T * (d // 2)), c["angle"].reshape(-1))


@pytest.mark.parametrize("idx", range(12))
def test_exact_oracle_encoder_matches_reference(golden, idx):
    """The correctly rounded C oracle == reference except admissible ties."""
    c = case(golden, f"enc{idx}")
    T, d, m, n, lay = (int(v) for v in c["cfg"])
    s16 = exact.scales(c["keys"], n, lay)
    assert np.array_equal(s16.view(np.uint16), c["scales"])
    a, r, clamped = exact.encode(c["keys"], s16, m, n, lay)
    compare_codes(c["keys"], lay, m, n, s16, a, r, c["angle"], c["radius"], exact=False)
    assert exact.pack(c["angle"], m) == c["angle_stream"].tobytes()
    assert exact.pack(c["radius"], n) == c["radius_stream"].tobytes()
    assert clamped == int(c["clamped"])


def test_adjacent_kat(golden):
    """SURVEY 8(c) extra KAT: ADJACENT m4n4 on 2 tokens."""
    c = case(golden, "kat_adjacent")
    s16 = po.scales_fp16(c["keys"], 4, po.ADJACENT)
    assert np.array_equal(s16.view(np.uint16), c["scales"])
    a, r, _ = po.encode_block(c["keys"], s16, 4, 4, po.ADJACENT)
    assert a.tolist() == [[10, 0, 8, 0], [12, 0, 8, 4]] == c["angle"].tolist()
    assert r.tolist() == [[15, 0, 0, 15], [6, 0, 15, 15]] == c["radius"].tolist()


@pytest.mark.parametrize("idx", range(6))
def test_oracle_cache_replay_matches_reference(golden, same_host_features, idx):
    c = case(golden, f"cache{idx}")
    T, d, m, n, lay, res = (int(v) for v in c["cfg"])
    oc = po.OracleCache(m, n, lay, res)
    oc.prefill(c["keys"], c["values"])
    for q, ref in zip(c["queries"], c["pre_scores"]):
        got = oc.scores(q)
        if same_host_features:
            assert np.array_equal(got, ref)
    for k, v in zip(c["app_keys"], c["app_values"]):
        oc.append(k, v)
    assert np.array_equal(oc.s16.view(np.uint16), c["scales"])
    a, r = oc.codes()
    if same_host_features:
        assert po.pack(a, m) == c["angle_stream"].tobytes()
        assert po.pack(r, n) == c["radius_stream"].tobytes()
    assert oc.clamps == int(c["clamps"])
    assert np.array_equal(oc.residual_keys(), c["residual_keys"])
    assert np.array_equal(po.radius_levels(oc.s16, n), c["radius_table"])
    assert np.array_equal(po.dequantize(a, r, oc.s16, m, lay)[:64], c["decoded"])
    temp = 1.0 / math.sqrt(d)
    for g, q in enumerate(c["queries"]):
        sc = oc.scores(q)
        if same_host_features:
            assert np.array_equal(sc, c["scores"][g])
        w = po.softmax64(sc, temp)
        np.testing.assert_allclose(w, c["weights"][g], rtol=0, atol=1e-15)
        np.testing.assert_allclose(po.attend(w, oc.all_values()), c["out"][g], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("idx", range(6))
def test_exact_oracle_scores_match_reference(golden, idx):
    """C LUT scorer on the reference's codes reproduces qk_scores bit-for-bit."""
    c = case(golden, f"cache{idx}")
    T, d, m, n, lay, res = (int(v) for v in c["cfg"])
    count = c["angle_stream"].size * 8 // m
    tq = (c["scores"].shape[1] - c["residual_keys"].shape[0])
    a = po.unpack(c["angle_stream"].tobytes(), m, tq * (d // 2)).reshape(tq, d // 2)
    r = po.unpack(c["radius_stream"].tobytes(), n, tq * (d // 2)).reshape(tq, d // 2)
    assert count >= tq * (d // 2)
    s16 = c["scales"].view(np.float16)
    for g, q in enumerate(c["queries"]):
        got = exact.lut_scores(q, a, r, s16, m, n, lay)
        assert np.array_equal(got, c["scores"][g][:tq])


@pytest.mark.parametrize("m", range(1, 9))
def test_tables_match_reference(golden, m):
    c = case(golden, f"table{m}")
    cs, sn = po.angle_unit_table(m)
    assert np.array_equal(cs, c["cos"]) and np.array_equal(sn, c["sin"])
    assert np.array_equal(po.query_table(c["q"], m, po.HALF_SPLIT), c["lut"])


def test_case_listing(golden):
    assert case_names(golden, "enc") == [f"enc{i}" for i in range(12)]
    assert case_names(golden, "cache") == [f"cache{i}" for i in range(6)]


@pytest.fixture(scope="module")
def golden_values():
    from pathlib import Path

    data = np.load(Path(__file__).resolve().parent / "golden" / "golden_values.npz")
    return {k: data[k] for k in data.files}


@pytest.mark.parametrize("idx", range(4))
def test_value_quantizer_matches_reference(golden_values, idx):
    """Per-token uniform value codes (the PackedKVCache quantize_values mode):
    codes, zero points, scales and dequantized rows bit-identical to the
    reference's quantize_uniform / dequantize_uniform / values()."""
    g = {k.split("/", 1)[1]: v for k, v in golden_values.items() if k.startswith(f"v{idx}/")}
    codes, zp, sc = po.quantize_values(g["values"], int(g["bits"]))
    assert np.array_equal(codes, g["codes"])
    assert np.array_equal(zp.view(np.uint32), g["zero_point"].view(np.uint32))
    assert np.array_equal(sc.view(np.uint32), g["scale"].view(np.uint32))
    deq = po.dequantize_values(codes, zp, sc)
    assert np.array_equal(deq.view(np.uint32), g["dequant"].view(np.uint32))
    assert np.array_equal(deq.view(np.uint32), g["cache_values"].view(np.uint32))
