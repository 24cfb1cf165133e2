"""HP-2 parity on the GPU: LUT scores bit-identical to the reference's fp32
sequence, float64 weights, and fused softmax.V within the stated tolerance."""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import paper_2502_00527_b200 as pq
from oracle import exact, polar_oracle as po
from tests.helpers import case, peak_close

pytestmark = pytest.mark.gpu

LAY = {0: pq.PairingLayout.ADJACENT, 1: pq.PairingLayout.HALF_SPLIT}

# Tolerances (stated):
#   quantized-token scores: bit-identical (same fp32 op sequence as qk_scores)
#   residual-token scores:  |err| <= 1e-5 * max(1, peak)  (fp32 dot, order differs from BLAS)
#   attention out fp32:     |err| <= 1e-4 * max(1, max|o|)
#   attention out bf16:     |err| <= 2^-7 * max|o| + one bf16 ulp
OUT_RTOL_F32 = 1e-4


def _replay(c):
    T, d, m, n, lay, res = (int(v) for v in c["cfg"])
    cache = pq.PackedKVCache(pq.QuantConfig(m, n, LAY[lay]), res)
    cache.prefill(c["keys"], c["values"])
    return cache, (T, d, m, n, lay, res)


@pytest.mark.parametrize("idx", range(6))
def test_golden_cache_scores_and_attention(golden, idx):
    c = case(golden, f"cache{idx}")
    cache, (T, d, m, n, lay, res) = _replay(c)
    for q, ref in zip(c["queries"], c["pre_scores"]):
        _check_scores(pq.qk_scores(q, cache), ref, cache)
    for k, v in zip(c["app_keys"], c["app_values"]):
        cache.append(k, v)
    assert np.array_equal(cache.scales.values.view(np.uint16), c["scales"])
    assert cache.clamp_events == int(c["clamps"])
    assert np.array_equal(cache.residual_keys, c["residual_keys"])
    assert np.array_equal(cache.radius_table(), c["radius_table"])
    snap = cache.quantized
    tq = cache.quantized_tokens
    ga = po.unpack(snap.angle_stream, m, tq * (d // 2)).reshape(tq, -1)
    gr = po.unpack(snap.radius_stream, n, tq * (d // 2)).reshape(tq, -1)
    ra = po.unpack(c["angle_stream"].tobytes(), m, tq * (d // 2)).reshape(tq, -1)
    rr = po.unpack(c["radius_stream"].tobytes(), n, tq * (d // 2)).reshape(tq, -1)
    tie = (ga != ra) | (gr != rr)
    assert tie.mean() <= 1e-4
    np.testing.assert_array_equal(cache.decode_quantized()[:64][~tie[:64].any(axis=1)],
                                  c["decoded"][~tie[:64].any(axis=1)])
    temp = 1.0 / math.sqrt(d)
    for g, q in enumerate(c["queries"]):
        sc = pq.qk_scores(q, cache)
        _check_scores(sc, c["scores"][g], cache, tie_rows=tie.any(axis=1))
        w = pq.attention_weights(sc, temp)
        np.testing.assert_allclose(w.sum(), 1.0, atol=1e-12)
        if not tie.any():
            # residual-token scores are fp32 dots whose summation order differs
            # from BLAS (1e-5 peak-relative); quantized-only weights match to rounding
            rtol = 1e-10 if cache.residual_tokens == 0 else 2e-5
            np.testing.assert_allclose(w, c["weights"][g], rtol=rtol, atol=1e-15)
        o = pq.decode_attention(q, cache)
        peak_close(o, c["out"][g], OUT_RTOL_F32)
    np.testing.assert_array_equal(cache.values(), np.concatenate([c["values"], c["app_values"]]))


def _check_scores(got, ref, cache, tie_rows=None):
    tq = cache.quantized_tokens
    assert got.shape == ref.shape and got.dtype == np.float32
    rows = np.ones(tq, bool) if tie_rows is None else ~tie_rows
    assert np.array_equal(got[:tq][rows], ref[:tq][rows]), "quantized-token scores must be bit-identical"
    if got.shape[0] > tq:
        peak_close(got[tq:], ref[tq:], 1e-5)


def test_reference_lut_tests():
    """test_lut_decode.py KATs through the GPU API."""
    t1 = pq.build_angle_table(1)
    assert np.allclose(t1.unit_vectors(), [[-1.0, 0.0], [1.0, 0.0]], atol=1e-6)
    t2 = pq.build_angle_table(2)
    assert np.allclose(t2.cos, [-1.0, 0.0, 1.0, 0.0], atol=1e-7)
    assert np.allclose(t2.sin, [0.0, -1.0, 0.0, 1.0], atol=1e-7)
    lut = pq.build_query_lut(np.array([1.0, 0.0]), t2, pq.PairingLayout.ADJACENT)
    assert np.allclose(lut.partial[0], t2.cos, atol=1e-7)
    keys = pq.KeyTensor(np.array([[0.0, 3.0], [0.0, 2.0]], np.float32), layout=pq.PairingLayout.ADJACENT)
    cache = pq.PackedKVCache(pq.QuantConfig(3, 2, pq.PairingLayout.ADJACENT), 0)
    cache.prefill(keys)
    a, r = cache.code_arrays()
    assert a.ravel().tolist() == [6, 6] and r.ravel().tolist() == [3, 2]
    assert np.allclose(pq.qk_scores(np.array([0.0, 1.0], np.float32), cache), [3.0, 2.0], atol=1e-5)
    z = pq.PackedKVCache(pq.QuantConfig(4, 4), 0)
    z.prefill(po.synthetic_keys(32, 8, seed=0))
    assert np.array_equal(pq.qk_scores(np.zeros(8, np.float32), z), np.zeros(32, np.float32))
    with pytest.raises(ValueError):
        pq.qk_scores(np.zeros(4, np.float32), z)
    with pytest.raises(ValueError):
        pq.attention_weights(np.zeros(0), 1.0)
    w = pq.attention_weights(np.full(4, 0.7), 0.5)
    assert np.allclose(w, 0.25)


@pytest.mark.parametrize("m,n", [(4, 4), (3, 2), (2, 2), (4, 2), (2, 4), (3, 4), (5, 3), (8, 8)])
@pytest.mark.parametrize("G", [1, 4, 8])
def test_batched_decode_vs_oracle(m, n, G):
    """Config-1 head shape (d=128, HALF_SPLIT), several units, bf16 V, GQA group G."""
    U, T = 4, 4096
    keys = np.stack([po.synthetic_keys(T, 128, seed=200 + u, outliers=(0, 1)) for u in range(U)])
    rng = np.random.default_rng(9)
    vals = torch.from_numpy(rng.standard_normal((U, T, 128)).astype(np.float32)).to(torch.bfloat16)
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(m, n), U, 128, 0, capacity=T + 1, page_tokens=128, shuffle_pages=True)
    cache.prefill(torch.from_numpy(keys).cuda(), vals.cuda())
    out = cache.decode(torch.from_numpy(q).cuda()).cpu().numpy()
    scores = cache.scores(torch.from_numpy(q).cuda()).cpu().numpy()
    v64 = vals.float().numpy().astype(np.float64)
    for u in range(U):
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        for g in range(G):
            ref = exact.lut_scores(q[u, g], a, r, s16, m, n, 1)
            assert np.array_equal(scores[u, g], ref)
            w = po.softmax64(ref, 1.0 / math.sqrt(128))
            peak_close(out[u, g], w @ v64[u], OUT_RTOL_F32)


def test_scores_into_caller_buffer():
    """UnitView.scores(out=...) (the bench's scores-only mode) writes the same
    bit-exact rows as the allocating call; bad buffers are rejected."""
    U, T, G = 3, 1000, 4
    keys = np.stack([po.synthetic_keys(T, 128, seed=500 + u) for u in range(U)])
    q = torch.from_numpy(np.random.default_rng(5).standard_normal((U, G, 128)).astype(np.float32)).cuda()
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 0, capacity=T)
    cache.prefill(torch.from_numpy(keys).cuda())
    ref = cache.scores(q)
    view = cache.view(0, U)
    buf = torch.full((U, G, T + 24), 7.0, dtype=torch.float32, device="cuda")  # wider rows: ld = T + 24
    got = view.scores(q, max_tokens=T, out=buf)
    assert got.data_ptr() == buf.data_ptr()
    assert torch.equal(got, ref)
    assert bool((buf[:, :, T:] == 7.0).all())  # nothing written past max_tokens
    with pytest.raises(ValueError):
        view.scores(q, max_tokens=T, out=buf.to(torch.float16))
    with pytest.raises(ValueError):
        view.scores(q, max_tokens=T, out=torch.empty((G, U, T), device="cuda").transpose(0, 1))
    with pytest.raises(ValueError):
        view.scores(q, max_tokens=T, out=buf[:, :, : T - 1])
    # a tile bound below the longest unit would cut its tokens (and overrun score rows)
    with pytest.raises(ValueError, match="max_tokens"):
        view.scores(q, max_tokens=T - 1)
    with pytest.raises(ValueError, match="max_tokens"):
        view.decode(q, max_tokens=T - 64)


@pytest.mark.parametrize("T,res", [(32768, 0), (9000, 64), (33, 32), (1, 1), (65, 0)])
def test_split_and_residual(T, res):
    """Long contexts (many splits), residual windows, tiny / ragged lengths."""
    U, G = 2, 4
    keys = np.stack([po.synthetic_keys(T, 128, seed=300 + u) for u in range(U)])
    rng = np.random.default_rng(T)
    vals = rng.standard_normal((U, T, 128)).astype(np.float32)
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, res, capacity=T + 1, value_dtype=torch.bfloat16)
    cache.prefill(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda())
    out = cache.decode(torch.from_numpy(q).cuda()).cpu().numpy()
    sc = cache.scores(torch.from_numpy(q).cuda()).cpu().numpy()
    vb = torch.from_numpy(vals).to(torch.bfloat16).float().numpy().astype(np.float64)
    for u in range(U):
        oc = po.OracleCache(4, 4, 1, res)
        oc.s16 = cache.scales16[u].cpu().numpy()
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        resid = keys[u][T - min(res, T):] if res else np.zeros((0, 128), np.float32)
        for g in range(G):
            ref = po.lut_scores(q[u, g], a, r, oc.s16, 4, 4, 1, resid)
            tq = a.shape[0]
            assert np.array_equal(sc[u, g, :tq], ref[:tq])
            if T > tq:
                peak_close(sc[u, g, tq:], ref[tq:], 1e-5)
            w = po.softmax64(ref, 1.0 / math.sqrt(128))
            peak_close(out[u, g], w @ vb[u], OUT_RTOL_F32)


def test_bf16_output_and_generic_group():
    """G=3 takes the generic kernel; bf16 output within 2^-7 relative."""
    U, T, G = 3, 2000, 3
    keys = np.stack([po.synthetic_keys(T, 128, seed=400 + u) for u in range(U)])
    rng = np.random.default_rng(1)
    vals = rng.standard_normal((U, T, 128)).astype(np.float32)
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(3, 2), U, 128, 0, capacity=T)
    cache.prefill(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda())
    o32 = cache.decode(torch.from_numpy(q).cuda()).cpu().numpy()
    o16 = cache.decode(torch.from_numpy(q).cuda(), out_dtype=torch.bfloat16).float().cpu().numpy()
    vb = torch.from_numpy(vals).to(torch.bfloat16).float().numpy().astype(np.float64)
    for u in range(U):
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        for g in range(G):
            ref = po.softmax64(exact.lut_scores(q[u, g], a, r, s16, 3, 2, 1), 1 / math.sqrt(128)) @ vb[u]
            peak_close(o32[u, g], ref, OUT_RTOL_F32)
            assert np.abs(o16[u, g] - ref).max() <= 2**-7 * np.abs(ref).max() + 2**-8 * np.abs(ref).max()


def test_append_stream_matches_oracle():
    """Streaming appends (K5) with frozen scales: codes, clamps and attention
    track the oracle cache token by token."""
    T, d, s = 200, 128, 16
    keys = po.synthetic_keys(T, d, seed=1)
    more = po.synthetic_keys(300, d, seed=2) * 1.3  # some radii outgrow the scales
    rng = np.random.default_rng(0)
    vals = rng.standard_normal((T + 300, d)).astype(np.float32)
    cache = pq.PackedKVCache(pq.QuantConfig(4, 4), s)
    cache.prefill(keys, vals[:T])
    oc = po.OracleCache(4, 4, 1, s)
    oc.prefill(keys, vals[:T])
    q = rng.standard_normal(d).astype(np.float32)
    for i, k in enumerate(more):
        cache.append(k, vals[T + i])
        oc.append(k, vals[T + i])
        if i % 50 == 49:
            ea, er, _ = exact.encode(np.concatenate([keys, more])[: cache.quantized_tokens], oc.s16, 4, 4, 1)
            a, r = cache.code_arrays()
            assert np.array_equal(a, ea) and np.array_equal(r, er)
            sc = pq.qk_scores(q, cache)
            ref = po.lut_scores(q, a, r, oc.s16, 4, 4, 1, oc.residual_keys())
            assert np.array_equal(sc[: a.shape[0]], ref[: a.shape[0]])
    assert cache.clamp_events == oc.clamps > 0
    assert cache.num_tokens == T + 300 and cache.residual_tokens == s


def test_state_errors():
    cache = pq.PackedKVCache(pq.QuantConfig(4, 4), 2)
    with pytest.raises(RuntimeError):
        cache.append(np.zeros(16, np.float32))
    with pytest.raises(RuntimeError):
        _ = cache.scales
    with pytest.raises(ValueError):
        cache.prefill(np.zeros((0, 16), np.float32))
    cache.prefill(po.synthetic_keys(10, 16, seed=0))
    with pytest.raises(RuntimeError):
        cache.prefill(po.synthetic_keys(4, 16, seed=0))
    with pytest.raises(ValueError):
        cache.append(np.zeros(8, np.float32))
    bad = pq.PackedKVCache(pq.QuantConfig(4, 4), 0)
    with pytest.raises(ValueError):
        bad.prefill(np.full((4, 16), np.nan, np.float32))
    assert not bad.prefilled


def test_views_and_workspace_reuse():
    """Per-layer views (the benchmark's launch pattern) equal the full-cache
    decode, and one view's workspace survives calls of different shapes
    (the fused split merge leaves its counters zeroed)."""
    L, upl, T = 3, 5, 3000
    U = L * upl
    keys = np.stack([po.synthetic_keys(T, 128, seed=900 + u) for u in range(U)])
    rng = np.random.default_rng(5)
    vals = torch.from_numpy(rng.standard_normal((U, T, 128)).astype(np.float32)).to(torch.bfloat16)
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 0, capacity=T)
    for layer in range(L):  # fill layer by layer through unit_start
        sl = slice(layer * upl, (layer + 1) * upl)
        cache.prefill(torch.from_numpy(keys[sl]).cuda(), vals[sl].cuda(), unit_start=layer * upl)
    assert cache.prefilled
    q4 = torch.from_numpy(rng.standard_normal((U, 4, 128)).astype(np.float32)).cuda()
    full = cache.decode(q4).cpu().numpy()
    view = cache.view(upl, 2 * upl)
    for rep in range(3):
        got = view.decode(q4[upl:2 * upl]).cpu().numpy()
        np.testing.assert_allclose(got, full[upl:2 * upl], rtol=0, atol=1e-6)
        q8 = torch.from_numpy(rng.standard_normal((upl, 8, 128)).astype(np.float32)).cuda()
        o8 = view.decode(q8, max_tokens=T).cpu().numpy()
        o8b = view.decode(q8, max_tokens=T, splits=7).cpu().numpy()  # different work split, same view
        np.testing.assert_allclose(o8, o8b, rtol=0, atol=2e-6)
        vb = vals.float().numpy().astype(np.float64)
        for u in range(upl):
            a, r = (t.cpu().numpy() for t in cache.code_arrays(upl + u))
            s16 = cache.scales16[upl + u].cpu().numpy()
            ref = po.softmax64(exact.lut_scores(q8[u, 3].cpu().numpy(), a, r, s16, 4, 4, 1), 1 / math.sqrt(128))
            peak_close(o8[u, 3], ref @ vb[upl + u], OUT_RTOL_F32)


@pytest.mark.parametrize("m,n", [(4, 4), (3, 2), (2, 2), (4, 2), (2, 4), (3, 4)])
@pytest.mark.parametrize("G", [4, 8])
@pytest.mark.parametrize("lay,res", [(1, 0), (0, 0), (1, 40)])
def test_dq_decode_vs_oracle(m, n, G, lay, res):
    """Dequantize + tensor-core scoring kernel (decode_dq.cu): fused output
    within the fp32 tolerance of softmax64(exact LUT scores) . V, both layouts,
    residual windows, ragged lengths."""
    U = 3
    lens = [3000, 1777, 33]
    T = max(lens)
    keys = [po.synthetic_keys(t, 128, seed=700 + u, outliers=(0, 1), layout=lay) for u, t in enumerate(lens)]
    rng = np.random.default_rng(m * 10 + n + G)
    vals = [rng.standard_normal((t, 128)).astype(np.float32) for t in lens]
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(m, n, LAY[lay]), U, 128, res, capacity=T + 1)
    for u in range(U):
        cache.prefill(torch.from_numpy(keys[u]).cuda().unsqueeze(0), torch.from_numpy(vals[u]).cuda().unsqueeze(0),
                      unit_start=u)
    qd = torch.from_numpy(q).cuda()
    out = cache.decode(qd, flags=pq._lib.PQB_DECODE_DQ).cpu().numpy()
    lut = cache.decode(qd, flags=pq._lib.PQB_DECODE_LUT).cpu().numpy()
    for u in range(U):
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        vb = torch.from_numpy(vals[u]).to(torch.bfloat16).float().numpy().astype(np.float64)
        t_u = lens[u]
        resid = keys[u][t_u - min(res, t_u):] if res else np.zeros((0, 128), np.float32)
        for g in range(G):
            ref = po.lut_scores(q[u, g], a, r, s16, m, n, lay, resid)
            o_ref = po.softmax64(ref, 1.0 / math.sqrt(128)) @ vb
            peak_close(out[u, g], o_ref, OUT_RTOL_F32)
            peak_close(lut[u, g], o_ref, OUT_RTOL_F32)
    if G == 8:  # the default fused path for G = 8 is the DQ kernel
        assert np.array_equal(cache.decode(qd).cpu().numpy(), out)


def test_dq_extreme_scales_and_zero_query():
    """Q' normalisation (2^e) with tiny / huge channel scales, dead channels and
    an all-zero query row."""
    U, T, G = 2, 700, 8
    rng = np.random.default_rng(3)
    keys = rng.standard_normal((U, T, 128)).astype(np.float32)
    keys[0] *= 1e-3
    keys[1] *= 300.0
    keys[:, :, 5] = 0.0
    keys[:, :, 69] = 0.0  # pair 5 dead in HALF_SPLIT -> scale 0
    vals = rng.standard_normal((U, T, 128)).astype(np.float32)
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    q[1, 2] = 0.0
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 0, capacity=T)
    cache.prefill(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda())
    out = cache.decode(torch.from_numpy(q).cuda(), flags=pq._lib.PQB_DECODE_DQ).cpu().numpy()
    for u in range(U):
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        vb = torch.from_numpy(vals[u]).to(torch.bfloat16).float().numpy().astype(np.float64)
        for g in range(G):
            ref = exact.lut_scores(q[u, g], a, r, s16, 4, 4, 1)
            peak_close(out[u, g], po.softmax64(ref, 1.0 / math.sqrt(128)) @ vb, OUT_RTOL_F32)


# ---------------------------------------------------------------- 4-bit values


def _vq4_cache(m, n, lay, res, lens, G, seed, shuffle=False, bits=4):
    U = len(lens)
    T = max(lens)
    keys = [po.synthetic_keys(t, 128, seed=seed + u, outliers=(0, 1), layout=lay) for u, t in enumerate(lens)]
    rng = np.random.default_rng(seed)
    vals = [rng.standard_normal((t, 128)).astype(np.float32) for t in lens]
    for v in vals:  # constant rows (scale 0) and a wide one
        v[min(3, len(v) - 1)] = 0.25
        v[len(v) // 2] *= 50.0
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(m, n, LAY[lay]), U, 128, res, capacity=T + 8, value_bits=bits,
                            shuffle_pages=shuffle)
    for u in range(U):
        cache.prefill(torch.from_numpy(keys[u]).cuda().unsqueeze(0), torch.from_numpy(vals[u]).cuda().unsqueeze(0),
                      unit_start=u)
    return cache, keys, vals, q


def _vq4_check(cache, keys, vals, q, m, n, lay, res, lens, outs, tol=OUT_RTOL_F32, bits=4):
    for u, t_u in enumerate(lens):
        codes, zp, sc = po.quantize_values(vals[u], bits)
        deq = po.dequantize_values(codes, zp, sc)
        got = cache.values_f32(u).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), deq.view(np.uint32))  # values() bit-identical
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        resid = keys[u][t_u - min(res, t_u):] if res else np.zeros((0, 128), np.float32)
        for g in range(q.shape[1]):
            ref = po.lut_scores(q[u, g], a, r, s16, m, n, lay, resid)
            o_ref = po.softmax64(ref, 1.0 / math.sqrt(128)) @ deq.astype(np.float64)
            for out in outs:
                peak_close(out[u, g], o_ref, tol)


@pytest.mark.parametrize("m,n", [(4, 4), (3, 2), (2, 4)])
@pytest.mark.parametrize("G", [4, 8])
@pytest.mark.parametrize("lay,res", [(1, 0), (0, 40)])
def test_vq4_decode_vs_oracle(m, n, G, lay, res):
    """4-bit per-token values (PackedKVCache(quantize_values=True)) read inside
    the DQ kernel: values() bit-identical to the reference quantizer (pinned by
    tests/golden/golden_values.npz), fused output within the fp32 tolerance of
    softmax64(LUT scores) . values(); the generic kernel agrees."""
    lens = [3000, 1777, 33]
    cache, keys, vals, q = _vq4_cache(m, n, lay, res, lens, G, seed=900 + 10 * m + n, shuffle=True)
    qd = torch.from_numpy(q).cuda()
    out = cache.decode(qd).cpu().numpy()
    gen = cache.decode(qd, flags=pq._lib.PQB_DECODE_FORCE_GENERIC).cpu().numpy()
    _vq4_check(cache, keys, vals, q, m, n, lay, res, lens, [out, gen])


def test_vq4_append_and_bf16_out():
    """Streaming append into 4-bit value pages (nibbles OR-ed into the tile
    words), G = 1 (generic kernel) and bf16 output."""
    lens = [500, 257]
    m, n, lay, res = 4, 4, 1, 16
    cache, keys, vals, q = _vq4_cache(m, n, lay, res, lens, 4, seed=77)
    rng = np.random.default_rng(5)
    for _ in range(40):
        k_new = rng.standard_normal((2, 128)).astype(np.float32)
        v_new = rng.standard_normal((2, 128)).astype(np.float32)
        cache.append(torch.from_numpy(k_new).cuda(), torch.from_numpy(v_new).cuda())
        for u in range(2):
            keys[u] = np.concatenate([keys[u], k_new[u:u + 1]])
            vals[u] = np.concatenate([vals[u], v_new[u:u + 1]])
    lens = [len(v) for v in vals]
    qd = torch.from_numpy(q).cuda()
    out = cache.decode(qd).cpu().numpy()
    out1 = np.stack([cache.decode(qd[:, g:g + 1]).cpu().numpy()[:, 0] for g in range(4)], axis=1)
    _vq4_check(cache, keys, vals, q, m, n, lay, res, lens, [out, out1])
    ob = cache.decode(qd, out_dtype=torch.bfloat16).float().cpu().numpy()
    peak_close(ob, out, 2.0 ** -7)


@pytest.mark.parametrize("bits", [2, 8])
@pytest.mark.parametrize("m,n", [(4, 4), (3, 2), (2, 4)])
@pytest.mark.parametrize("G", [4, 8])
@pytest.mark.parametrize("lay,res", [(1, 0), (0, 40)])
def test_vq2_vq8_decode_vs_oracle(bits, m, n, G, lay, res):
    """2- and 8-bit per-token values (kv_cache.py:206-207 with value_bits 2 / 8)
    as code pages read inside the DQ kernel (m4n4, m3n2; other shapes by the
    generic kernel): values() bit-identical to the reference quantizer, fused
    output within the fp32 tolerance of softmax64(LUT scores) . values()."""
    lens = [3000, 1777, 33]
    cache, keys, vals, q = _vq4_cache(m, n, lay, res, lens, G, seed=500 + bits + 10 * m + n, shuffle=True,
                                      bits=bits)
    qd = torch.from_numpy(q).cuda()
    out = cache.decode(qd).cpu().numpy()
    gen = cache.decode(qd, flags=pq._lib.PQB_DECODE_FORCE_GENERIC).cpu().numpy()
    lin = cache._all().decode(qd, flags=pq._lib.PQB_DECODE_DQ | pq._lib.PQB_DECODE_DQ_LINEAR).cpu().numpy()
    _vq4_check(cache, keys, vals, q, m, n, lay, res, lens, [out, gen, lin], bits=bits)


@pytest.mark.parametrize("bits", [2, 8])
def test_vq2_vq8_append(bits):
    lens = [500, 257]
    m, n, lay, res = 4, 4, 1, 16
    cache, keys, vals, q = _vq4_cache(m, n, lay, res, lens, 4, seed=79, bits=bits)
    rng = np.random.default_rng(6)
    for _ in range(40):
        k_new = rng.standard_normal((2, 128)).astype(np.float32)
        v_new = rng.standard_normal((2, 128)).astype(np.float32)
        cache.append(torch.from_numpy(k_new).cuda(), torch.from_numpy(v_new).cuda())
        for u in range(2):
            keys[u] = np.concatenate([keys[u], k_new[u:u + 1]])
            vals[u] = np.concatenate([vals[u], v_new[u:u + 1]])
    lens = [len(v) for v in vals]
    out = cache.decode(torch.from_numpy(q).cuda()).cpu().numpy()
    _vq4_check(cache, keys, vals, q, m, n, lay, res, lens, [out], bits=bits)


def test_vq4_rejects_other_widths():
    with pytest.raises(ValueError):
        pq.PolarKVCache(pq.QuantConfig(4, 4), 1, 128, 0, value_bits=3)
    with pytest.raises(ValueError):
        pq.PolarKVCache(pq.QuantConfig(4, 4), 1, 64, 0, value_bits=4)


@pytest.mark.parametrize("page_tokens", [32, 64, 256, 512])
@pytest.mark.parametrize("G", [4, 8])
def test_dq_page_sizes(page_tokens, G):
    """The decode kernel's per-warp tile cursor (page, tile-in-page advanced by
    8 tiles per step) for 1, 2, 8 and 16 tiles per page, shuffled page tables,
    ragged lengths that end mid-page."""
    lens = [5000, 1057, 70]
    U = len(lens)
    keys = [po.synthetic_keys(t, 128, seed=40 + u, outliers=(0, 1)) for u, t in enumerate(lens)]
    rng = np.random.default_rng(page_tokens + G)
    vals = [rng.standard_normal((t, 128)).astype(np.float32) for t in lens]
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 0, capacity=max(lens) + 1, page_tokens=page_tokens,
                            shuffle_pages=True)
    for u in range(U):
        cache.prefill(torch.from_numpy(keys[u]).cuda().unsqueeze(0), torch.from_numpy(vals[u]).cuda().unsqueeze(0),
                      unit_start=u)
    qd = torch.from_numpy(q).cuda()
    out = cache.decode(qd).cpu().numpy()
    # regression: at G = 8 the end-of-segment merge scratch once overran warp
    # 0's mbarriers (CTAs whose later segments issue TMA: the short third unit)
    lut = cache.decode(qd, flags=pq._lib.PQB_DECODE_LUT).cpu().numpy()
    scores = cache.scores(qd).cpu().numpy()  # bit-exact qk_scores sequence, every page size
    for u in range(U):
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        vb = torch.from_numpy(vals[u]).to(torch.bfloat16).float().numpy().astype(np.float64)
        for g in range(G):
            ref = po.lut_scores(q[u, g], a, r, s16, 4, 4, 1, np.zeros((0, 128), np.float32))
            ex = exact.lut_scores(q[u, g], a, r, s16, 4, 4, 1)
            assert np.array_equal(scores[u, g, :lens[u]].view(np.uint32), ex.view(np.uint32))
            o_ref = po.softmax64(ref, 1.0 / math.sqrt(128)) @ vb
            peak_close(out[u, g], o_ref, OUT_RTOL_F32)
            peak_close(lut[u, g], o_ref, OUT_RTOL_F32)


@pytest.mark.parametrize("m,n", [(4, 4), (3, 2), (2, 4), (4, 2)])
@pytest.mark.parametrize("G", [4, 8])
@pytest.mark.parametrize("T,res,page", [(4096, 0, 256), (1000, 64, 64), (33, 32, 32), (70, 0, 128)])
def test_dq_scores_mode(m, n, G, T, res, page):
    """Scores-only calls with PQB_DECODE_DQ (the tensor-core contraction, SURVEY
    8(c) tolerance) against the bit-exact LUT rows: max|d| <= 1e-4 max(1, peak)
    per (unit, query) row, residual windows and ragged tails included."""
    U = 3
    keys = np.stack([po.synthetic_keys(T, 128, seed=700 + u, outliers=(0, 1)) for u in range(U)])
    rng = np.random.default_rng(T + G)
    q = torch.from_numpy(rng.standard_normal((U, G, 128)).astype(np.float32)).to(torch.bfloat16).cuda()
    cache = pq.PolarKVCache(pq.QuantConfig(m, n), U, 128, res, capacity=T, page_tokens=page, shuffle_pages=True)
    cache.prefill(torch.from_numpy(keys).cuda())
    view = cache.view(0, U)
    exact_rows = view.scores(q).cpu().numpy()
    fast = view.scores(q, flags=pq._lib.PQB_DECODE_DQ).cpu().numpy()
    assert fast.shape == exact_rows.shape == (U, G, T)
    for u in range(U):
        for g in range(G):
            tol = 1e-4 * max(1.0, float(np.abs(exact_rows[u, g]).max()))
            err = float(np.abs(fast[u, g] - exact_rows[u, g]).max())
            assert err <= tol, (u, g, err, tol)


@pytest.mark.parametrize("G", [4, 8])
@pytest.mark.parametrize("T", [70, 4096, 20000])
def test_separate_merge_kernel_matches_in_kernel_merge(G, T):
    """PQB_DECODE_MERGE_KERNEL (split merge in its own PDL launch) gives the
    in-kernel merge's outputs bit for bit (same LSE sequence per element)."""
    U = 5
    keys = np.stack([po.synthetic_keys(T, 128, seed=900 + u) for u in range(U)])
    rng = np.random.default_rng(T)
    vals = torch.from_numpy(rng.standard_normal((U, T, 128)).astype(np.float32)).to(torch.bfloat16)
    q = torch.from_numpy(rng.standard_normal((U, G, 128)).astype(np.float32)).cuda()
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 0, capacity=T, value_dtype=torch.bfloat16)
    cache.prefill(torch.from_numpy(keys).cuda(), vals.cuda())
    for dt in (torch.float32, torch.bfloat16):
        a = cache.decode(q, out_dtype=dt)
        b = cache.decode(q, out_dtype=dt, flags=pq._lib.PQB_DECODE_MERGE_KERNEL)
        assert torch.equal(a, b)


def test_decode_launch_count_policy():
    """pqb_decode_launches: the split merge gets its own launch for G = 8 from
    16K tokens and whenever units span more than 8 segments, never with
    NO_COMBINE; a merge-kernel shape still decodes to the LUT path's outputs."""
    lib = pq._lib.load()
    assert lib.pqb_decode_launches(128, 4, 32768, 0) == 1  # configs[1] layer
    # configs[0]: a short launch, on 8-CTA clusters (one launch); without them 16+ segments per unit
    assert lib.pqb_decode_launches(8, 4, 4096, 0) == 1
    assert lib.pqb_decode_launches(8, 4, 4096, pq._lib.PQB_DECODE_NO_CLUSTER) == 2
    # the cluster path needs m = n = 4 with bf16 values; other stores keep the merge launch
    bf16, vq4 = pq._lib.PQB_BF16, pq._lib.PQB_VQ4
    assert lib.pqb_decode_launches_ex(32, 8, 32768, 0, 4, 4, bf16) == 1
    assert lib.pqb_decode_launches_ex(32, 8, 32768, 0, 3, 2, bf16) == 2
    assert lib.pqb_decode_launches_ex(32, 8, 32768, 0, 4, 4, vq4) == 2
    # configs[3] layer: the thread-block-cluster path (4 CTAs per unit, DSMEM merge) on B200, one launch;
    # without it the split merge gets its own launch
    assert lib.pqb_decode_launches(32, 8, 32768, 0) == 1
    assert lib.pqb_decode_launches(32, 8, 32768, pq._lib.PQB_DECODE_NO_CLUSTER) == 2
    assert lib.pqb_decode_launches(32, 8, 4096, 0) == 1
    assert lib.pqb_decode_launches(128, 4, 32768, pq._lib.PQB_DECODE_MERGE_KERNEL) == 2
    assert lib.pqb_decode_launches(8, 4, 4096, pq._lib.PQB_DECODE_NO_COMBINE) == 1
    assert lib.pqb_decode_launches(8, 1, 4096, 0) == 1  # LUT kernel: merge in-kernel


@pytest.mark.parametrize("G", [4, 8])
@pytest.mark.parametrize("values", ["bf16", "f32", "vq4"])
def test_dq_split_shapes(G, values):
    """The DQ kernel's persistent work split (decode_dq.cu): ragged units cut at
    CTA counts from one CTA to a few tiles per CTA, so CTA ranges start and end
    inside units, cover several whole units and run past a unit's last tile
    (many merge segments per unit).  Outputs within
    the fp32 tolerance of softmax64(exact scores) . V at every split, the
    separate merge launch bit-identical to the in-kernel merge, and the fast
    shared-memory layout in use."""
    lens = [1, 33, 700, 64, 2000, 5, 129, 1024]
    U, T, res = len(lens), max(lens), 8
    rng = np.random.default_rng(G * 7 + len(values))
    keys = [po.synthetic_keys(t, 128, seed=1300 + u, outliers=(0, 1)) for u, t in enumerate(lens)]
    vals = [rng.standard_normal((t, 128)).astype(np.float32) for t in lens]
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    vkw = dict(value_bits=4) if values == "vq4" else dict(value_dtype=torch.float32 if values == "f32" else torch.bfloat16)
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, res, capacity=T + 1, page_tokens=64, **vkw)
    for u in range(U):
        cache.prefill(torch.from_numpy(keys[u]).cuda().unsqueeze(0), torch.from_numpy(vals[u]).cuda().unsqueeze(0),
                      unit_start=u)
    refs = []
    for u in range(U):
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        vv = cache.values_f32(u).cpu().numpy().astype(np.float64)
        resid = keys[u][lens[u] - min(res, lens[u]):]
        refs.append([po.softmax64(po.lut_scores(q[u, g], a, r, s16, 4, 4, 1, resid), 1.0 / math.sqrt(128)) @ vv
                     for g in range(G)])
    qd = torch.from_numpy(q).cuda()
    for splits in (1, 2, 3, 5, 13, 40, 148):
        out = cache.decode(qd, splits=splits).cpu().numpy()
        sep = cache.decode(qd, splits=splits, flags=pq._lib.PQB_DECODE_MERGE_KERNEL).cpu().numpy()
        assert np.array_equal(out, sep), splits
        for u in range(U):
            for g in range(G):
                peak_close(out[u, g], refs[u][g], OUT_RTOL_F32)
    assert pq._lib.load().pqb_decode_dq_layout() == 1  # the product table at its fixed address


@pytest.mark.parametrize("G,U,T", [(8, 32, 8192), (4, 32, 8192), (4, 64, 8192)])
def test_dq_cluster_merge(G, U, T):
    """The thread-block-cluster path (units x k CTAs fill the GPU, k = 4 or 8:
    each unit's CTAs form a cluster and LSE-merge their partials through
    distributed shared memory): outputs within the fp32 tolerance of the oracle
    on sampled units, one launch per call, and within fp32 round-off of the
    non-cluster path."""
    lib = pq._lib.load()
    assert lib.pqb_decode_launches(U, G, T, 0) == 1
    rng = np.random.default_rng(U + G)
    keys = np.stack([po.synthetic_keys(T, 128, seed=2100 + u, outliers=(0, 1)) for u in range(U)])
    vals = rng.standard_normal((U, T, 128)).astype(np.float32)
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 0, capacity=T, page_tokens=256, value_dtype=torch.bfloat16)
    cache.prefill(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda())
    qd = torch.from_numpy(q).cuda()
    out = cache.decode(qd).cpu().numpy()
    for _ in range(5):  # deterministic: the stage rings and the DSMEM merge leave no ordering to chance
        assert np.array_equal(cache.decode(qd).cpu().numpy(), out)
    alt = cache.decode(qd, flags=pq._lib.PQB_DECODE_NO_CLUSTER).cpu().numpy()
    for u in (0, 1, U // 2, U - 1):
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        vb = torch.from_numpy(vals[u]).to(torch.bfloat16).float().numpy().astype(np.float64)
        for g in range(G):
            ref = po.softmax64(po.lut_scores(q[u, g], a, r, s16, 4, 4, 1), 1.0 / math.sqrt(128)) @ vb
            peak_close(out[u, g], ref, OUT_RTOL_F32)
    np.testing.assert_allclose(out, alt, rtol=0, atol=1e-5 * max(1.0, float(np.abs(alt).max())))


def test_dq_cluster_merge_ragged_residual():
    """Cluster path with ragged units (some CTAs of a cluster past their unit's
    last tile) and a residual window: within the fp32 tolerance of the oracle."""
    U, G, res, T = 32, 8, 16, 8192
    lens = [T if u % 3 else max(40, (u * 997) % T) for u in range(U)]
    assert pq._lib.load().pqb_decode_launches(U, G, T, 0) == 1
    rng = np.random.default_rng(77)
    keys = [po.synthetic_keys(t, 128, seed=2300 + u, outliers=(0, 1)) for u, t in enumerate(lens)]
    vals = [rng.standard_normal((t, 128)).astype(np.float32) for t in lens]
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, res, capacity=T + 1, page_tokens=256,
                            value_dtype=torch.bfloat16)
    for u in range(U):
        cache.prefill(torch.from_numpy(keys[u]).cuda().unsqueeze(0), torch.from_numpy(vals[u]).cuda().unsqueeze(0),
                      unit_start=u)
    out = cache.decode(torch.from_numpy(q).cuda(), max_tokens=T).cpu().numpy()
    for u in (0, 3, 6, 7, 30):
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        vb = torch.from_numpy(vals[u]).to(torch.bfloat16).float().numpy().astype(np.float64)
        resid = keys[u][lens[u] - min(res, lens[u]):]
        for g in range(G):
            ref = po.softmax64(po.lut_scores(q[u, g], a, r, s16, 4, 4, 1, resid), 1.0 / math.sqrt(128)) @ vb
            peak_close(out[u, g], ref, OUT_RTOL_F32)


@pytest.mark.parametrize("G", [4, 8])
def test_dq_balanced_split(G):
    """The cost-balanced persistent split (CTA ranges of >= 192 tiles, so the
    balancing is active: a range crossing into a second unit is shortened) at
    several CTA counts: outputs within the fp32 tolerance of the oracle, and the
    in-launch and separate-launch split merges bit-identical."""
    lens = [20000, 13000, 20000, 7001, 16384]
    U, T = len(lens), max(lens)
    rng = np.random.default_rng(40 + G)
    keys = [po.synthetic_keys(t, 128, seed=1700 + u, outliers=(0, 1)) for u, t in enumerate(lens)]
    vals = [rng.standard_normal((t, 128)).astype(np.float32) for t in lens]
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, 0, capacity=T, page_tokens=256, value_dtype=torch.bfloat16)
    for u in range(U):
        cache.prefill(torch.from_numpy(keys[u]).cuda().unsqueeze(0), torch.from_numpy(vals[u]).cuda().unsqueeze(0),
                      unit_start=u)
    refs = []
    for u in range(U):
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        vb = torch.from_numpy(vals[u]).to(torch.bfloat16).float().numpy().astype(np.float64)
        refs.append([po.softmax64(po.lut_scores(q[u, g], a, r, s16, 4, 4, 1), 1.0 / math.sqrt(128)) @ vb
                     for g in range(G)])
    qd = torch.from_numpy(q).cuda()
    for splits in (3, 7, 11):
        out = cache.decode(qd, splits=splits, flags=pq._lib.PQB_DECODE_MERGE_INKERNEL).cpu().numpy()
        sep = cache.decode(qd, splits=splits, flags=pq._lib.PQB_DECODE_MERGE_KERNEL).cpu().numpy()
        assert np.array_equal(out, sep), splits
        for u in range(U):
            for g in range(G):
                peak_close(out[u, g], refs[u][g], OUT_RTOL_F32)


@pytest.mark.parametrize("m,n", [(4, 4), (3, 2), (2, 4), (3, 4)])
@pytest.mark.parametrize("G", [4, 8])
@pytest.mark.parametrize("lay,res,page", [(1, 0, 256), (0, 40, 64), (1, 16, 32)])
def test_f32_values_dq_vs_oracle(m, n, G, lay, res, page):
    """The reference's default value cache (fp32 rows, kv_cache.py:8-9, :209)
    in the DQ kernel (one 18 KB stage per warp, fp32 P.V on the CUDA cores):
    fp32 output within 1e-4 of softmax64(LUT scores) . V with the exact fp32
    values; the linear-layout build and the generic kernel agree."""
    lens = [3000, 1777, 33]
    U, T = len(lens), max(lens)
    keys = [po.synthetic_keys(t, 128, seed=300 + u, outliers=(0, 1), layout=lay) for u, t in enumerate(lens)]
    rng = np.random.default_rng(m * 100 + n * 10 + G)
    vals = [rng.standard_normal((t, 128)).astype(np.float32) * 3 for t in lens]
    q = rng.standard_normal((U, G, 128)).astype(np.float32)
    cache = pq.PolarKVCache(pq.QuantConfig(m, n, LAY[lay]), U, 128, res, capacity=T + 1, page_tokens=page,
                            value_dtype=torch.float32, shuffle_pages=True)
    for u in range(U):
        cache.prefill(torch.from_numpy(keys[u]).cuda().unsqueeze(0), torch.from_numpy(vals[u]).cuda().unsqueeze(0),
                      unit_start=u)
    qd = torch.from_numpy(q).cuda()
    outs = [cache.decode(qd).cpu().numpy(),
            cache._all().decode(qd, flags=pq._lib.PQB_DECODE_DQ | pq._lib.PQB_DECODE_DQ_LINEAR).cpu().numpy(),
            cache._all().decode(qd, flags=pq._lib.PQB_DECODE_FORCE_GENERIC).cpu().numpy()]
    for u in range(U):
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        s16 = cache.scales16[u].cpu().numpy()
        resid = keys[u][lens[u] - min(res, lens[u]):] if res else np.zeros((0, 128), np.float32)
        v64 = vals[u].astype(np.float64)
        for g in range(G):
            ref = po.lut_scores(q[u, g], a, r, s16, m, n, lay, resid)
            o_ref = po.softmax64(ref, 1.0 / math.sqrt(128)) @ v64
            for o in outs:
                peak_close(o[u, g], o_ref, OUT_RTOL_F32)
