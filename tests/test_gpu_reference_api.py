"""The reference's element-wise functions, tables, qk_scores_direct and the
snapshot import on the GPU, against fixtures made by the unmodified reference
(tests/golden/make_golden_api.py, tests/golden/make_golden.py) and the
reference's own tests (test_polar_codec.py:40-148, test_lut_decode.py:41-77,
test_acceptance.py:43-92, test_kv_cache.py:207-241)."""

from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

import paper_2502_00527_b200 as pq
from oracle import polar_oracle as po
from tests.helpers import case

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "golden_api.npz"
TWO_PI = 2 * math.pi


@pytest.fixture(scope="module")
def gapi():
    data = np.load(GOLD)
    return {k: data[k] for k in data.files}


def circular_distance(a, b):
    d = np.abs(np.asarray(a) - np.asarray(b)) % TWO_PI
    return np.minimum(d, TWO_PI - d)


# ------------------------------------------------------------------ to_polar


def test_to_polar_f64_matches_reference(gapi):
    x, y = gapi["polar_f64/x"], gapi["polar_f64/y"]
    r, t = pq.to_polar(x, y)
    assert r.dtype == np.float64 and t.dtype == np.float64
    # libm vs CUDA double hypot / atan2: both within 1-2 ulp of the true value
    np.testing.assert_allclose(r, gapi["polar_f64/r"], rtol=4e-16, atol=0)
    assert np.abs(t - gapi["polar_f64/t"]).max() <= 8 * np.spacing(TWO_PI)
    assert np.all((t >= 0) & (t < TWO_PI))


def test_to_polar_f32_matches_reference(gapi):
    """Radius bit-identical (glibc hypotf order); angle = the correctly rounded
    pipeline, which differs from numpy's SIMD arctan2 by at most a few ulp."""
    x, y = gapi["polar_f32/x"], gapi["polar_f32/y"]
    r, t = pq.to_polar(x, y)
    assert r.dtype == np.float32 and t.dtype == np.float32
    assert np.array_equal(r.view(np.uint32), gapi["polar_f32/r"].view(np.uint32))
    ref_t = gapi["polar_f32/t"]
    ulps = np.abs(t.view(np.int32).astype(np.int64) - ref_t.view(np.int32).astype(np.int64))
    wrap = np.minimum(np.abs(t - ref_t), TWO_PI - np.abs(t - ref_t)) <= 4 * np.spacing(np.float32(TWO_PI))
    assert np.all((ulps <= 4) | wrap), int(ulps.max())  # numpy's SIMD arctan2: ~1 ulp off on ~1/6 of inputs
    assert np.all((t >= 0) & (t < np.float32(TWO_PI)))


def test_to_polar_examples():
    """test_polar_codec.py:40-49."""
    r, t = pq.to_polar(0.0, 2.0)
    assert np.isclose(r, 2.0) and np.isclose(t, 1.5 * math.pi)
    r, t = pq.to_polar(-1.0, 0.0)
    assert np.isclose(r, 1.0) and t == 0.0  # 2 pi wraps to 0
    r, t = pq.to_polar(0.0, 0.0)
    assert r == 0.0 and np.isclose(t, math.pi)
    r, t = pq.to_polar(np.float32([3.0]), np.float32(4.0))  # broadcast, float32 kept
    assert r.dtype == np.float32 and r.shape == (1,) and r[0] == 5.0


# ------------------------------------------------------------ quantize_angle


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_quantize_angle_matches_reference(gapi, prec):
    th = gapi[f"qa_{prec}/theta"]
    for m in range(1, 9):
        got = pq.quantize_angle(th, m)
        assert got.dtype == np.uint8
        assert np.array_equal(got, gapi[f"qa_{prec}/codes"][m - 1]), m


def test_quantize_angle_examples_and_bounds():
    """test_polar_codec.py:66-99 and acceptance C1 (test_acceptance.py:43-61)."""
    assert pq.quantize_angle(1.5 * math.pi, 3) == 6
    for m in range(1, 9):
        assert pq.quantize_angle(0.0, m) == 0
        assert pq.quantize_angle(TWO_PI - 1e-9, m) == 0
    assert pq.quantize_angle(math.pi / 4, 2) == 0 and pq.quantize_angle(3 * math.pi / 4, 2) == 2
    rng = np.random.default_rng(101)
    theta = rng.uniform(0, TWO_PI, 120_000)
    for m in (1, 2, 3, 4, 6, 8):
        codes = pq.quantize_angle(theta, m)
        decoded = (pq.angle_grid(m)[codes] + math.pi) % TWO_PI
        assert circular_distance(theta, decoded).max() <= math.pi / 2**m + 1e-6
        shifted = (theta + TWO_PI) % TWO_PI
        assert np.array_equal(codes, pq.quantize_angle(shifted, m))
    assert np.allclose(pq.angle_grid(2), [-math.pi, -math.pi / 2, 0.0, math.pi / 2])
    with pytest.raises(ValueError):
        pq.quantize_angle(0.0, 9)


def test_angle_grid_matches_reference(gapi):
    for m in range(1, 9):
        assert np.array_equal(pq.angle_grid(m), gapi[f"grid/m{m}"])


# ----------------------------------------------------------- quantize_radius


@pytest.mark.parametrize("i", range(4))
def test_quantize_radius_matches_reference(gapi, i):
    from paper_2502_00527_b200.codec import quantize_radius_counted

    rad, sc, bits = gapi[f"qr{i}/radius"], gapi[f"qr{i}/scale"], int(gapi[f"qr{i}/bits"])
    codes, clamped = quantize_radius_counted(rad, sc, bits)
    assert np.array_equal(np.asarray(codes), gapi[f"qr{i}/codes"])
    assert clamped == int(gapi[f"qr{i}/clamped"])


def test_quantize_radius_examples_and_bound():
    """test_polar_codec.py:133-148 and acceptance C1's radius half."""
    assert pq.quantize_radius(np.float32(2.2), np.float32(1.0), 2) == 2
    assert pq.quantize_radius(np.float32(0.0), np.float32(1.0), 2) == 0
    assert pq.quantize_radius(np.float32(9.9), np.float32(1.0), 2) == 3
    assert pq.quantize_radius(np.float32(5.0), np.float32(0.0), 2) == 0
    rng = np.random.default_rng(101)
    radii = rng.uniform(0, 37.5, 120_000).astype(np.float32)
    for n in (1, 2, 3, 4, 8):
        scale = np.float16(radii.max() / (2**n - 1)).astype(np.float32)
        codes = pq.quantize_radius(radii, scale, n)
        err = np.abs(radii.astype(np.float64) - codes.astype(np.float64) * float(scale))
        assert err.max() <= float(scale) / 2 + 1e-6


# ---------------------------------------------------------------- tables


@pytest.mark.parametrize("m", range(1, 9))
def test_tables_replay_golden(golden, m):
    """build_angle_table / build_query_lut bit-identical to the reference's
    (lut_decode.py:63-104; golden table{m} fixtures)."""
    c = case(golden, f"table{m}")
    t = pq.build_angle_table(m)
    assert np.array_equal(t.cos.view(np.uint32), c["cos"].view(np.uint32))
    assert np.array_equal(t.sin.view(np.uint32), c["sin"].view(np.uint32))
    lut = pq.build_query_lut(c["q"], t, pq.PairingLayout.HALF_SPLIT)
    assert np.array_equal(lut.partial.view(np.uint32), c["lut"].view(np.uint32))


def test_lut_kats():
    """test_lut_decode.py:52-77: antipodal table symmetry, LUT basis rows, q = 0."""
    for m in range(1, 9):
        t = pq.build_angle_table(m)
        h = 1 << (m - 1)
        assert np.allclose(t.cos[:h], -t.cos[h:], atol=1e-6) and np.allclose(t.sin[:h], -t.sin[h:], atol=1e-6)
    t = pq.build_angle_table(3)
    lut = pq.build_query_lut(np.array([0.0, 1.0, 1.0, 0.0], np.float32), t, pq.PairingLayout.ADJACENT)
    assert np.array_equal(lut.partial[0], t.sin) and np.array_equal(lut.partial[1], t.cos)
    z = pq.build_query_lut(np.zeros(8, np.float32), t)
    assert not z.partial.any()


# ------------------------------------------------------ qk_scores_direct


def test_qk_scores_direct_matches_reference(gapi):
    m, n, lay, res = (int(v) for v in gapi["direct/cfg"])
    cache = pq.PackedKVCache(pq.QuantConfig(m, n, pq.PairingLayout(lay)), res)
    cache.prefill(gapi["direct/keys"])
    q = gapi["direct/q"]
    got = pq.qk_scores_direct(q, cache)
    ref = gapi["direct/scores"]
    assert got.dtype == np.float32 and got.shape == ref.shape
    peak = max(1.0, float(np.abs(ref).max()))
    assert np.abs(got - ref).max() <= 1e-5 * peak  # two fp32 dot orders
    lut = pq.qk_scores(q, cache)
    assert np.abs(lut - got).max() <= 1e-4 * peak  # acceptance C2's LUT == dequant tolerance
    counter = pq.OpCounter()
    pq.qk_scores_direct(q, cache, counter)
    tq, tr = cache.quantized_tokens, cache.residual_tokens
    assert counter.lookups == 3 * tq * 64 and counter.multiplies == 2 * tq * 128 + tr * 128


# ------------------------------------------------------------- snapshots


def test_load_snapshot_keeps_streaming(gapi, tmp_path):
    """A reference-written snapshot loads into the paged GPU cache, and two
    further appends give exactly the reference's loaded-cache state
    (test_kv_cache.py:207-223)."""
    p = tmp_path / "ref.snap"
    p.write_bytes(gapi["snap/blob"].tobytes())
    cache = pq.load_snapshot(p)
    assert cache.prefilled and cache.residual_len == 4
    from paper_2502_00527_b200 import container

    snap = container.parse_snapshot(p.read_bytes())
    assert cache.quantized.angle_stream == snap.codes.angle_stream
    assert cache.quantized.radius_stream == snap.codes.radius_stream
    assert np.array_equal(cache.residual_keys, snap.residual_keys)
    assert cache.clamp_events == snap.clamp_events
    out = tmp_path / "ours.snap"
    pq.save_snapshot(cache, out)
    assert out.read_bytes() == p.read_bytes()
    for row in gapi["snap/app_keys"]:
        cache.append(row)
    q = cache.quantized
    assert q.angle_stream == gapi["snap/after_angle"].tobytes()
    assert q.radius_stream == gapi["snap/after_radius"].tobytes()
    assert np.array_equal(cache.residual_keys, gapi["snap/after_residual"])
    assert cache.clamp_events == int(gapi["snap/after_clamps"])
    assert cache.num_tokens == int(gapi["snap/after_tokens"])
    assert not cache.values().any()  # values come back as zeros


def test_snapshot_round_trip_through_gpu_cache(tmp_path):
    """test_kv_cache.py:207-241: save -> load -> identical state; nothing-quantized case."""
    keys = po.synthetic_keys(300, 128, seed=3, outliers=(0, 1))
    cache = pq.PackedKVCache(pq.QuantConfig(3, 2), 16)
    cache.prefill(keys)
    for row in po.synthetic_keys(20, 128, seed=4):
        cache.append(row)
    p = tmp_path / "c.snap"
    pq.save_snapshot(cache, p)
    loaded = pq.load_snapshot(p)
    assert loaded.quantized == cache.quantized
    assert loaded.scales.values.tobytes() == cache.scales.values.tobytes()
    assert np.array_equal(loaded.residual_keys, cache.residual_keys)
    assert loaded.clamp_events == cache.clamp_events and loaded.residual_len == 16
    q = np.random.default_rng(0).standard_normal(128).astype(np.float32)
    assert np.array_equal(pq.qk_scores(q, loaded), pq.qk_scores(q, cache))
    loaded.append(po.synthetic_keys(1, 128, seed=9)[0])
    assert loaded.num_tokens == cache.num_tokens + 1
    small = pq.PackedKVCache(pq.QuantConfig(), 8)
    small.prefill(po.synthetic_keys(3, 16, seed=1))
    pq.save_snapshot(small, p)
    assert pq.load_snapshot(p).quantized_tokens == 0


def test_import_unit_into_batched_cache():
    """PolarKVCache.import_unit: a unit restored from its snapshot decodes like the original."""
    import torch

    U, T = 3, 2000
    keys = np.stack([po.synthetic_keys(T, 128, seed=60 + u, outliers=(0, 1)) for u in range(U)])
    vals = torch.randn(U, T, 128).to(torch.bfloat16)
    src = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 32, capacity=T, page_tokens=128)
    src.prefill(torch.from_numpy(keys).cuda(), vals.cuda())
    dst = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 32, capacity=T, page_tokens=128, shuffle_pages=True)
    for u in range(U):
        s = src.snapshot_unit(u)
        dst.import_unit(u, s.codes, s.scales, s.residual_keys, s.clamp_events, values=vals[u].cuda())
    assert dst.prefilled
    q = torch.randn(U, 4, 128, device="cuda")
    assert torch.equal(dst.decode(q), src.decode(q))
    for u in range(U):
        assert dst.export_codes(u) == src.export_codes(u)
