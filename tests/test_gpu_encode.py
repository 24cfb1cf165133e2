"""HP-1 parity on the GPU: scales bit-exact, codes bit-exact vs the correctly
rounded C oracle and tie-bounded vs the reference (golden fixtures / numpy
oracle), across layouts, bit widths, dtypes, vector and generic kernels."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2502_00527_b200 as pq
from oracle import exact, polar_oracle as po
from tests.helpers import case, compare_codes

pytestmark = pytest.mark.gpu

LAY = {0: pq.PairingLayout.ADJACENT, 1: pq.PairingLayout.HALF_SPLIT}


@pytest.mark.parametrize("idx", range(12))
def test_golden_encoder(golden, idx):
    c = case(golden, f"enc{idx}")
    T, d, m, n, lay = (int(v) for v in c["cfg"])
    cfg = pq.QuantConfig(m, n, LAY[lay])
    s = pq.compute_radius_scales(c["keys"], cfg)
    assert s.values.dtype == np.float16
    assert np.array_equal(s.values.view(np.uint16), c["scales"])
    codes = pq.encode_keys(c["keys"], s, cfg)
    a, r = codes.angle_codes(), codes.radius_codes()
    compare_codes(c["keys"], lay, m, n, s.values, a, r, c["angle"], c["radius"], exact=False)
    ea, er, _ = exact.encode(c["keys"], s.values, m, n, lay)
    assert np.array_equal(a, ea) and np.array_equal(r, er)
    assert codes.angle_stream == exact.pack(ea, m) and codes.radius_stream == exact.pack(er, n)
    assert len(codes.angle_stream) == pq.stream_bytes(T * (d // 2), m)


def test_adjacent_kat(golden):
    c = case(golden, "kat_adjacent")
    cfg = pq.QuantConfig(4, 4, pq.PairingLayout.ADJACENT)
    s = pq.compute_radius_scales(c["keys"], cfg)
    assert np.array_equal(s.values.view(np.uint16), c["scales"])
    codes = pq.encode_keys(c["keys"], s, cfg)
    assert codes.angle_codes().tolist() == [[10, 0, 8, 0], [12, 0, 8, 4]]
    assert codes.radius_codes().tolist() == [[15, 0, 0, 15], [6, 0, 15, 15]]


# ---- reference unit KATs (test_polar_codec.py) replayed through the GPU API


def test_scales_examples():
    keys = np.array([[1.0, 0.0], [2.0, 0.0], [3.0, 0.0]], dtype=np.float32)
    s = pq.compute_radius_scales(keys, pq.QuantConfig(4, 2, pq.PairingLayout.ADJACENT))
    assert s.values.dtype == np.float16 and float(s.as_compute()[0]) == 1.0
    s = pq.compute_radius_scales(np.array([[7.0, 0.0]], np.float32), pq.QuantConfig(4, 3, pq.PairingLayout.ADJACENT))
    assert float(s.as_compute()[0]) == 1.0


def test_scales_zero_channel_and_empty():
    s = pq.compute_radius_scales(np.zeros((4, 2), np.float32), pq.QuantConfig(4, 4, pq.PairingLayout.ADJACENT))
    assert float(s.as_compute()[0]) == 0.0
    with pytest.raises(ValueError):
        pq.compute_radius_scales(np.zeros((0, 2), np.float32), pq.QuantConfig())


def test_scale_overflow_raises():
    keys = np.array([[60000.0 * 15, 0.0]], np.float32) * 10
    with pytest.raises(ValueError):
        pq.compute_radius_scales(keys, pq.QuantConfig(4, 4, pq.PairingLayout.ADJACENT))


def test_worked_example():
    keys = pq.KeyTensor(np.array([[0.0, 2.0]], np.float32), layout=pq.PairingLayout.ADJACENT)
    cfg = pq.QuantConfig(3, 2, pq.PairingLayout.ADJACENT)
    s = pq.ChannelScales(np.array([1.0]))
    codes = pq.encode_keys(keys, s, cfg)
    assert codes.angle_codes().tolist() == [[6]] and codes.radius_codes().tolist() == [[2]]
    assert np.allclose(pq.decode_keys(codes, s, cfg).data, [[0.0, 2.0]], atol=1e-6)


def test_zero_radius_decodes_to_origin():
    cfg = pq.QuantConfig(3, 2, pq.PairingLayout.ADJACENT)
    s = pq.ChannelScales(np.array([1.0]))
    for a in range(8):
        codes = pq.PolarCodes.from_arrays(np.array([[a]], np.uint8), np.array([[0]], np.uint8), cfg)
        assert np.array_equal(pq.decode_keys(codes, s).data, [[0.0, 0.0]])


def test_quantize_radius_and_angle_examples():
    """quantize_radius 2.2->2, 0->0, 9.9->3 (clamp), zero-scale->0 and the
    angle KATs (3pi/2 at m=3 -> 6; 2pi - eps wraps to 0) through encode_keys."""
    cfg = pq.QuantConfig(3, 2, pq.PairingLayout.ADJACENT)
    s = pq.ChannelScales(np.array([1.0, 0.0]))
    keys = np.array([[2.2, 0.0, 5.0, 5.0], [0.0, 0.0, 1.0, 0.0], [9.9, 0.0, 0.0, 0.0], [0.0, -3.0, 0.0, 0.0]],
                    np.float32)
    codes = pq.encode_keys(keys, s, cfg)
    r = codes.radius_codes()
    a = codes.angle_codes()
    assert r[:, 0].tolist() == [2, 0, 3, 3]
    assert r[:, 1].tolist() == [0, 0, 0, 0] and a[:, 1].tolist() == [0, 0, 0, 0]  # dead channel
    assert a[0, 0] == 4 and a[1, 0] == 4  # phi = 0 -> theta = pi -> code 2^(m-1); origin canonical
    assert a[3, 0] == 2  # phi = -pi/2 -> theta = pi/2 -> 2


def test_encode_decode_encode_identity():
    rng = np.random.default_rng(23)
    mat = rng.standard_normal((200, 16)).astype(np.float32)
    mat[:50] *= 1e-3
    mat[:, 3] = 0.0
    mat[:, 11] = 0.0
    cfg = pq.QuantConfig(4, 3)
    s = pq.compute_radius_scales(mat, cfg)
    first = pq.encode_keys(mat, s, cfg)
    second = pq.encode_keys(pq.decode_keys(first, s), s, cfg)
    assert first.angle_stream == second.angle_stream and first.radius_stream == second.radius_stream


def test_lattice_fixed_point():
    rng = np.random.default_rng(17)
    for m, n in [(2, 2), (4, 4), (3, 6), (8, 2)]:
        cfg = pq.QuantConfig(m, n)
        s = pq.ChannelScales(rng.uniform(0.05, 2.0, 8).astype(np.float32))
        angle = rng.integers(0, 2**m, (50, 8)).astype(np.uint8)
        radius = rng.integers(1, 2**n, (50, 8)).astype(np.uint8)
        codes = pq.PolarCodes.from_arrays(angle, radius, cfg)
        again = pq.encode_keys(pq.decode_keys(codes, s), s, cfg)
        assert np.array_equal(again.angle_codes(), angle) and np.array_equal(again.radius_codes(), radius)


def test_validation():
    cfg = pq.QuantConfig(4, 4)
    with pytest.raises(ValueError):
        pq.encode_keys(np.zeros((2, 8), np.float32), pq.ChannelScales(np.ones(3)), cfg)
    with pytest.raises(ValueError):
        pq.encode_keys(np.full((2, 8), np.inf, np.float32), pq.ChannelScales(np.ones(4)), cfg)
    with pytest.raises(ValueError):
        pq.compute_radius_scales(np.full((2, 8), np.nan, np.float32), cfg)


@pytest.mark.parametrize("bits", range(1, 9))
def test_pack_unpack_round_trip(bits):
    rng = np.random.default_rng(bits)
    for tokens, half in [(1, 1), (7, 3), (33, 5), (64, 64)]:
        a = rng.integers(0, 2**bits, (tokens, half)).astype(np.uint8)
        codes = pq.PolarCodes.from_arrays(a, a, pq.QuantConfig(bits, bits))
        assert codes.angle_stream == po.pack(a, bits)
        assert np.array_equal(codes.angle_codes(), a)


# ---- batched device path at config-1 and config-5 shapes vs the exact oracle


def _batched(keys_np: np.ndarray, cfg, dtype=torch.float32, page_tokens=128, shuffle=False):
    U, T, d = keys_np.shape
    cache = pq.PolarKVCache(cfg, U, d, 0, capacity=T + 1, page_tokens=page_tokens, shuffle_pages=shuffle)
    cache.prefill(torch.from_numpy(keys_np).to("cuda", dtype))
    return cache


@pytest.mark.parametrize("m,n", [(4, 4), (3, 2), (2, 2), (2, 4), (3, 4), (4, 2)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_batched_encode_vs_exact_oracle(m, n, dtype):
    T = 4096
    keys = np.stack([po.synthetic_keys(T, 128, seed=100 + u, outliers=(0, 1)) for u in range(4)])
    if dtype == torch.bfloat16:
        keys = torch.from_numpy(keys).to(torch.bfloat16).float().numpy()
    cache = _batched(keys, pq.QuantConfig(m, n), dtype=dtype, shuffle=True)
    for u in range(4):
        s16 = exact.scales(keys[u], n, 1)
        assert np.array_equal(cache.scales16[u].cpu().numpy().view(np.uint16), s16.view(np.uint16))
        a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
        ea, er, clamps = exact.encode(keys[u], s16, m, n, 1)
        assert np.array_equal(a, ea), np.argwhere(a != ea)[:5]
        assert np.array_equal(r, er)
        codes = cache.export_codes(u)
        assert codes.angle_stream == exact.pack(ea, m) and codes.radius_stream == exact.pack(er, n)
    assert int(cache.clamp_counts.sum()) == 0


def test_config5_sample_bit_exact():
    """Config 5 (bulk prefill encode) on a sampled slab: 4 (layer, head) units
    x 262144 tokens, every m in {2,3,4} x n in {2,4}, bf16 inputs."""
    T = 262144
    rng_keys = np.stack([po.synthetic_keys(T, 128, seed=500 + u, outliers=(0, 1)) for u in range(2)])
    keys16 = torch.from_numpy(rng_keys).to(torch.bfloat16)
    keys = keys16.float().numpy()
    for m in (2, 3, 4):
        for n in (2, 4):
            cache = pq.PolarKVCache(pq.QuantConfig(m, n), 2, 128, 0, capacity=T + 1, page_tokens=256)
            cache.prefill(keys16.cuda())
            for u in range(2):
                s16 = exact.scales(keys[u], n, 1)
                ea, er, _ = exact.encode(keys[u], s16, m, n, 1)
                a, r = (t.cpu().numpy() for t in cache.code_arrays(u))
                assert np.array_equal(a, ea) and np.array_equal(r, er), (m, n, u)


def test_generic_path_matches_vector_path():
    """Strided / odd-shaped inputs take the generic kernel; results must equal
    the vector kernel's on the same values."""
    keys = np.stack([po.synthetic_keys(1000, 128, seed=7 + u) for u in range(2)])
    cfg = pq.QuantConfig(4, 4)
    a = _batched(keys, cfg)
    big = torch.zeros((2, 1000, 136), dtype=torch.float32, device="cuda")
    big[:, :, 3:131] = torch.from_numpy(keys).cuda()
    b = pq.PolarKVCache(cfg, 2, 128, 0, capacity=1001)
    b.prefill(big[:, :, 3:131])  # misaligned rows -> generic kernels
    for u in range(2):
        assert torch.equal(a.scales16[u], b.scales16[u])
        for x, y in zip(a.code_arrays(u), b.code_arrays(u)):
            assert torch.equal(x, y)


@pytest.mark.parametrize("d", [2, 10, 16, 64, 256])
def test_odd_dims_vs_exact(d):
    keys = po.synthetic_keys(333, d, seed=d, layout=0)
    cfg = pq.QuantConfig(3, 5, pq.PairingLayout.ADJACENT)
    s = pq.compute_radius_scales(keys, cfg)
    assert np.array_equal(s.values.view(np.uint16), exact.scales(keys, 5, 0).view(np.uint16))
    codes = pq.encode_keys(keys, s, cfg)
    ea, er, _ = exact.encode(keys, s.values, 3, 5, 0)
    assert np.array_equal(codes.angle_codes(), ea) and np.array_equal(codes.radius_codes(), er)


def test_f16_inputs():
    keys = po.synthetic_keys(512, 128, seed=3).astype(np.float16)
    cfg = pq.QuantConfig(4, 4)
    cache = pq.PolarKVCache(cfg, 1, 128, 0, capacity=513)
    cache.prefill(torch.from_numpy(keys).cuda().unsqueeze(0))
    k32 = keys.astype(np.float32)
    s16 = exact.scales(k32, 4, 1)
    ea, er, _ = exact.encode(k32, s16, 4, 4, 1)
    a, r = (t.cpu().numpy() for t in cache.code_arrays(0))
    assert np.array_equal(a, ea) and np.array_equal(r, er)


def test_edge_points_take_exact_path():
    """Points exactly on / within an ulp of bin edges and at the axes."""
    m, n = 4, 4
    edges = (np.arange(16) + 0.5) * np.pi / 8 - np.pi
    eps = np.array([-2e-7, -1e-7, 0.0, 1e-7, 2e-7])
    phi = (edges[:, None] + eps[None, :]).reshape(-1)
    r = np.linspace(0.5, 3.0, phi.size)
    x = (r * np.cos(phi)).astype(np.float32)
    y = (r * np.sin(phi)).astype(np.float32)
    ax = np.array([0, 1, 0, -1, 0, -0.0, 1e-30, -1e-30], np.float32)
    ay = np.array([1, 0, -1, 0, 0, 1, 1, -1], np.float32)
    x, y = np.concatenate([x, ax]), np.concatenate([y, ay])
    pad = (-x.size) % 64
    x = np.concatenate([x, np.ones(pad, np.float32)]).reshape(-1, 64)
    y = np.concatenate([y, np.ones(pad, np.float32)]).reshape(-1, 64)
    for layout in (pq.PairingLayout.HALF_SPLIT, pq.PairingLayout.ADJACENT):
        keys = po.join_xy(x, y, layout.value)  # d = 128: the vector (fast-path) kernel
        for mm in (1, 2, 3, 4, 5, 6, 8):
            cfg = pq.QuantConfig(mm, n, layout)
            s = pq.ChannelScales(np.full(64, 0.25, np.float32))
            codes = pq.encode_keys(keys, s, cfg)
            ea, er, _ = exact.encode(keys, s.values, mm, n, layout.value)
            assert np.array_equal(codes.angle_codes(), ea), (layout, mm)
            assert np.array_equal(codes.radius_codes(), er)


@pytest.mark.parametrize("m", [1, 2, 3])
def test_exact_diagonal_ties(m):
    """|x| == |y| exactly (about 0.3% of bf16 pairs): the m = 2 bin edge; the
    fast path resolves these without the double-precision fallback."""
    rng = np.random.default_rng(11)
    v = torch.from_numpy(rng.standard_normal((2048, 64)).astype(np.float32)).to(torch.bfloat16).float().numpy()
    sx = rng.choice([-1.0, 1.0], size=v.shape).astype(np.float32)
    sy = rng.choice([-1.0, 1.0], size=v.shape).astype(np.float32)
    keys = np.concatenate([v * sx, v * sy], axis=1)  # HALF_SPLIT: x = dims[:64], y = dims[64:]
    keys[::7, 5] = 0.0  # a few axis points too
    cfg = pq.QuantConfig(m, 4)
    cache = pq.PolarKVCache(cfg, 1, 128, 0, capacity=keys.shape[0] + 1)
    cache.prefill(torch.from_numpy(keys).cuda().to(torch.bfloat16).unsqueeze(0))
    s16 = exact.scales(keys, 4, 1)
    ea, er, _ = exact.encode(keys, s16, m, 4, 1)
    a, r = (t.cpu().numpy() for t in cache.code_arrays(0))
    assert np.array_equal(a, ea) and np.array_equal(r, er)


def _encode_raw(keys: torch.Tensor, s16: np.ndarray, cfg, page_tokens: int, kernel: str):
    """K2 alone with given scales into a fresh shuffled paged cache; kernel
    'fast' (encode_fast.cu when the call qualifies) or 'v8' (forced)."""
    import os

    from paper_2502_00527_b200.codec import encode_device

    U, T, d = keys.shape
    cache = pq.PolarKVCache(cfg, U, d, 0, capacity=T + 1, page_tokens=page_tokens, shuffle_pages=True)
    cache.scales16.copy_(torch.from_numpy(s16.view(np.float16)).cuda())
    old = os.environ.pop("PQB_ENCODE_KERNEL", None)
    if kernel == "v8":
        os.environ["PQB_ENCODE_KERNEL"] = "v8"
    try:
        encode_device(keys, cache.scales16, cfg, cache.store_ref(), clamp_counts=cache.clamp_counts)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("PQB_ENCODE_KERNEL", None)
        if old is not None:
            os.environ["PQB_ENCODE_KERNEL"] = old
    cache.host_quant[:] = T
    return cache


def _hard_keys(U: int, T: int, seed: int) -> np.ndarray:
    """Synthetic keys plus the cases the fast path must route or resolve:
    bin-edge angles, exact diagonal ties, axis points, zero rows, a dead
    channel (scale 0), tiny and large magnitudes."""
    keys = np.stack([po.synthetic_keys(T, 128, seed=seed + u, outliers=(0, 1)) for u in range(U)])
    rng = np.random.default_rng(seed)
    # bin edges of every m in {2, 3, 4} (+- a few ulp) on channel pairs 10..13
    for j, m in zip(range(10, 13), (2, 3, 4)):
        k = rng.integers(0, 1 << m, size=(U, T))
        phi = (k + 0.5) * np.pi / (1 << (m - 1)) - np.pi + rng.choice([-2e-7, 0.0, 2e-7], size=(U, T))
        r = rng.uniform(0.2, 2.0, size=(U, T))
        keys[:, :, j], keys[:, :, 64 + j] = (r * np.cos(phi)).astype(np.float32), (r * np.sin(phi)).astype(np.float32)
    v = rng.standard_normal((U, T)).astype(np.float32)
    keys[:, :, 20], keys[:, :, 84] = v, -v  # |x| == |y|
    keys[:, ::5, 21] = 0.0  # axis points
    keys[:, ::13, 33] = 0.0
    keys[:, ::13, 97] = 0.0  # origin
    keys[:, :, 7] = 0.0
    keys[:, :, 71] = 0.0  # dead channel 7 -> scale 0
    keys[:, ::17, 40] *= 1e-12  # tiny
    return keys


@pytest.mark.parametrize("m,n", [(4, 4), (3, 2), (2, 4), (2, 2), (4, 2), (3, 4), (3, 3), (2, 3), (4, 3)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("layout", [1, 0])
def test_fast_encoder_vs_v8_and_exact(m, n, dtype, layout):
    """encode_fast.cu against the per-call-grid kernel and the exact C oracle:
    codes bit-identical, clamp counts equal (scales shrunk on a few channels so
    radii clamp), ragged T (partial 1024-token item and 32-token stage)."""
    U, T = 3, 2 * 1024 + 357
    keys_np = _hard_keys(U, T, seed=40 + m * 10 + n)
    keys = torch.from_numpy(keys_np).to(dtype)
    if layout == 0:  # ADJACENT: interleave the HALF_SPLIT halves
        keys = torch.stack([keys[..., :64], keys[..., 64:]], dim=-1).reshape(U, T, 128)
    keys_f = keys.float().numpy()
    cfg = pq.QuantConfig(m, n, LAY[layout])
    s16 = np.stack([exact.scales(keys_f[u], n, layout) for u in range(U)])
    s16 = s16.view(np.float16).copy()
    s16[:, 30:34] = (s16[:, 30:34].astype(np.float32) * 0.6).astype(np.float16)  # clamps
    fast = _encode_raw(keys.cuda(), s16.view(np.uint16), cfg, 128, "fast")
    ref = _encode_raw(keys.cuda(), s16.view(np.uint16), cfg, 128, "v8")
    assert torch.equal(fast.clamp_counts, ref.clamp_counts)
    assert int(fast.clamp_counts.sum()) > 0
    for u in range(U):
        fa, fr = fast.code_arrays(u)
        ra, rr = ref.code_arrays(u)
        assert torch.equal(fa, ra), np.argwhere((fa != ra).cpu().numpy())[:5]
        assert torch.equal(fr, rr)
        ea, er, clamps = exact.encode(keys_f[u], s16[u], m, n, layout)
        assert np.array_equal(fa.cpu().numpy(), ea) and np.array_equal(fr.cpu().numpy(), er)
        assert int(fast.clamp_counts[u]) == clamps


def test_fast_encoder_offset_fallback():
    """A start token that is not a multiple of 16 (the fast kernel's stage
    alignment) routes to encode_v8; the codes land at the offset unchanged."""
    from paper_2502_00527_b200.codec import encode_device

    keys = torch.from_numpy(_hard_keys(2, 700, seed=5)).to(torch.bfloat16).cuda()
    cfg = pq.QuantConfig(4, 4)
    kf = keys.float().cpu().numpy()
    s16 = np.stack([exact.scales(kf[u], 4, 1) for u in range(2)])
    a = _encode_raw(keys, s16, cfg, 64, "fast")
    b = pq.PolarKVCache(cfg, 2, 128, 0, capacity=800, page_tokens=64, shuffle_pages=True)
    b.scales16.copy_(a.scales16)
    encode_device(keys, b.scales16, cfg, b.store_ref(), tok_offset_const=8)
    torch.cuda.synchronize()
    b.host_quant[:] = 708
    for u in range(2):
        for x, y in zip(a.code_arrays(u), b.code_arrays(u)):
            assert torch.equal(x, y[8:])
