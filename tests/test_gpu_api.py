"""The reference's own cache / acceptance tests (test_kv_cache.py,
test_acceptance.py C2/C7/C9) replayed against the GPU package: the drop-in
check for PackedKVCache and the score paths."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2502_00527_b200 as pq
from oracle import polar_oracle as po

pytestmark = pytest.mark.gpu


def _keys(tokens, dim=16, seed=0, **kw):
    return pq.gen_synthetic_keys(pq.SyntheticConfig(tokens, dim, seed=seed, **kw))


def _cache(tokens=10, residual=3, dim=16, m=4, n=4, seed=0):
    cache = pq.PackedKVCache(pq.QuantConfig(m, n), residual)
    cache.prefill(_keys(tokens, dim, seed))
    return cache


def test_prefill_split_counts():
    c = _cache(tokens=10, residual=3)
    assert (c.quantized_tokens, c.residual_tokens, c.num_tokens) == (7, 3, 10)


def test_prefill_shorter_than_window():
    c = _cache(tokens=4, residual=8)
    assert c.quantized_tokens == 0 and c.residual_tokens == 4 and c.prefilled


def test_scales_match_offline():
    keys = _keys(20)
    c = pq.PackedKVCache(pq.QuantConfig(4, 4), 4)
    c.prefill(keys)
    assert c.scales.values.tobytes() == pq.compute_radius_scales(keys, c.cfg).values.tobytes()


def test_residual_holds_newest_exactly():
    keys = _keys(10)
    c = pq.PackedKVCache(pq.QuantConfig(4, 4), 3)
    c.prefill(keys)
    assert np.array_equal(c.residual_keys, keys.data[7:])


def test_append_zero_window_and_flush():
    c = _cache(tokens=5, residual=0)
    c.append(_keys(1, seed=9).data[0])
    assert (c.quantized_tokens, c.residual_tokens) == (6, 0)
    keys = _keys(3)
    c = pq.PackedKVCache(pq.QuantConfig(4, 4), 2)
    c.prefill(keys)
    extra = _keys(5, seed=7)
    for row in extra.data:
        c.append(row)
    assert (c.quantized_tokens, c.residual_tokens) == (6, 2)
    assert np.array_equal(c.residual_keys, extra.data[-2:])


def test_clamp_counter():
    cfg = pq.QuantConfig(4, 4, pq.PairingLayout.ADJACENT)
    c = pq.PackedKVCache(cfg, 0)
    c.prefill(np.array([[1.0, 0.0]], np.float32))
    assert c.clamp_events == 0
    c.append(np.array([2.0, 0.0], np.float32))
    assert c.clamp_events == 1
    assert c.code_arrays()[1][-1, 0] == 15
    keys = _keys(50, seed=3)
    c = pq.PackedKVCache(pq.QuantConfig(4, 4), 4)
    c.prefill(keys)
    for row in keys.data[:20]:
        c.append(row)
    assert c.clamp_events == 0


def test_decode_preserves_token_order():
    keys = _keys(30, seed=5)
    c = pq.PackedKVCache(pq.QuantConfig(6, 6), 4)
    c.prefill(keys)
    dec = c.decode_quantized()
    err = np.linalg.norm(dec - keys.data[:26], axis=1)
    shifted = np.linalg.norm(dec[1:] - keys.data[:25], axis=1)
    assert err.max() < 0.2 and np.median(shifted) > np.median(err[1:])


def test_bit_reports():
    c = pq.PackedKVCache(pq.QuantConfig(4, 4), 0)
    c.prefill(_keys(256, dim=128))
    r = c.memory_report()
    assert r.payload_bits == 131072 and r.payload_bits_per_element == 4.0
    c = pq.PackedKVCache(pq.QuantConfig(3, 5), 2)
    c.prefill(_keys(37, dim=10))
    codes = c.quantized
    packed = 8 * (len(codes.angle_stream) + len(codes.radius_stream))
    assert 0 <= packed - c.memory_report().payload_bits < 16
    c = pq.PackedKVCache(pq.QuantConfig(4, 4), 128)
    c.prefill(_keys(12200, dim=128, seed=1))
    assert abs(c.memory_report().avg_bits_per_element - 4.16) <= 0.05


def test_values_and_value_quant_mode():
    keys = _keys(6)
    values = np.arange(6 * 16, dtype=np.float32).reshape(6, 16)
    c = pq.PackedKVCache(pq.QuantConfig(4, 4), 2)
    c.prefill(keys, values)
    c.append(keys.data[0], values[0])
    out = c.values()
    assert out.shape == (7, 16) and np.array_equal(out[:6], values)
    v = np.linspace(-2, 2, 6 * 16, dtype=np.float32).reshape(6, 16)
    c = pq.PackedKVCache(pq.QuantConfig(4, 4), 2, quantize_values=True, value_bits=8)
    c.prefill(keys, v)
    out = c.values()
    assert not np.array_equal(out[:6], v) and np.allclose(out[:6], v, atol=2e-2)


def test_value_quant_mode_bit_exact_vs_reference_semantics():
    """Per-token uniform quantize->dequantize (baseline_quant.py:58-110, 167)."""
    rng = np.random.default_rng(4)
    for dim, bits in [(32, 2), (32, 4), (32, 8), (128, 2), (128, 4), (128, 8), (128, 3)]:
        # d = 128 with 2 / 4 / 8 bits: code pages read by the decode kernels
        v = rng.standard_normal((50, dim)).astype(np.float32)
        v[3] = 1.5  # constant row -> scale 0 -> exact zero-point
        c = pq.PackedKVCache(pq.QuantConfig(4, 4), 0, quantize_values=True, value_bits=bits)
        c.prefill(_keys(50, dim=dim), v)
        top = (1 << bits) - 1
        zp = v.min(axis=1, keepdims=True)
        scale = (v.max(axis=1, keepdims=True) - zp) / top
        with np.errstate(divide="ignore", invalid="ignore"):
            raw = np.rint((v - zp) / scale)
        raw = np.where(scale == 0.0, 0.0, raw)
        codes = np.clip(raw, 0, top).astype(np.uint8)
        ref = (codes.astype(np.float32) * scale + zp).astype(np.float32)
        assert np.array_equal(c.values(), ref)


def test_snapshot_stable_across_appends():
    c = _cache(tokens=10, residual=2)
    snap = c.snapshot()
    before = (snap.codes.num_tokens, snap.residual_keys.copy())
    for row in _keys(4, seed=6).data:
        c.append(row)
    assert snap.codes.num_tokens == before[0] and np.array_equal(snap.residual_keys, before[1])


def test_acceptance_c2_lut_equals_dequant():
    """C2 (test_acceptance.py:64-92), 120 instances: LUT scores == dequantize-then-dot
    within 1e-4 * peak over random m, n in [2, 8], residual {0, 16}, both layouts."""
    rng = np.random.default_rng(202)
    for i in range(120):
        tokens = int(np.exp(rng.uniform(math.log(16), math.log(4096))))
        m, n = int(rng.integers(2, 9)), int(rng.integers(2, 9))
        res = int(rng.choice([0, 0, 0, 16]))
        layout = pq.PairingLayout.HALF_SPLIT if i % 2 else pq.PairingLayout.ADJACENT
        keys = rng.standard_normal((tokens, 128)).astype(np.float32)
        keys[:, :16] *= 5.0
        c = pq.PackedKVCache(pq.QuantConfig(m, n, layout), res)
        c.prefill(keys)
        q = rng.standard_normal(128).astype(np.float32)
        lut = pq.qk_scores(q, c)
        direct = pq.qk_scores_direct(q, c)
        peak = max(1.0, float(np.abs(direct).max()))
        assert np.abs(lut - direct).max() <= 1e-4 * peak, i


def test_acceptance_c7_operation_counts():
    for tokens in (4096, 8192):
        c = pq.PackedKVCache(pq.QuantConfig(4, 4), 0)
        c.prefill(_keys(tokens, 128, seed=7))
        q = np.random.default_rng(tokens).standard_normal(128).astype(np.float32)
        a, b = pq.OpCounter(), pq.OpCounter()
        pq.qk_scores(q, c, a)
        pq.qk_scores_direct(q, c, b)
        assert a.multiplies == tokens * 64 + 128 * 16
        assert b.multiplies == 2 * tokens * 128
        assert a.additions == tokens * 64 + 64 * 16


def test_acceptance_c9_streaming_invariants():
    for residual_len in (0, 1, 64):
        for prefill_tokens in (1, 32, 200):
            pool = _keys(prefill_tokens, 16, seed=residual_len + prefill_tokens)
            c = pq.PackedKVCache(pq.QuantConfig(4, 4), residual_len)
            c.prefill(pool)
            appended = prefill_tokens
            history = list(pool.data)
            rng = np.random.default_rng(99)
            for _ in range(60):
                row = pool.data[int(rng.integers(0, prefill_tokens))]
                c.append(row)
                history.append(row)
                appended += 1
                assert c.num_tokens == appended
                assert c.residual_tokens == min(residual_len, appended)
            if c.residual_tokens:
                assert np.array_equal(c.residual_keys, np.stack(history[appended - c.residual_tokens:]))
            assert c.clamp_events == 0
            assert c.decode_quantized().shape[0] + c.residual_tokens == appended


def test_decode_attention_single_head_api():
    keys = po.synthetic_keys(500, 64, seed=3)
    rng = np.random.default_rng(3)
    vals = rng.standard_normal((500, 64)).astype(np.float32)
    c = pq.PackedKVCache(pq.QuantConfig(4, 4), 8)
    c.prefill(keys, vals)
    q = rng.standard_normal((3, 64)).astype(np.float32)
    out = pq.decode_attention(q, c)
    for g in range(3):
        w = pq.attention_weights(pq.qk_scores(q[g], c), 1 / 8)
        ref = w @ c.values().astype(np.float64)
        assert np.abs(out[g] - ref).max() <= 1e-4 * max(1.0, np.abs(ref).max())
    assert pq.decode_attention(q[0], c).shape == (64,)
