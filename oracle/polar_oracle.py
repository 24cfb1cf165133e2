"""CPU oracle for the PolarQuant hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (/root/reference/pkg/src/
polarquant), used solely as the checker in tests/, by __graft_entry__.smoke()
and by bench.py's cpu_baseline / --impl reference leg.  The product package
(paper_2502_00527_b200) never imports it.

It performs the same numpy float32/float64 operations in the same order as
the reference, so on a given host its outputs are the reference's outputs;
that is pinned by tests/test_oracle_golden.py against fixtures generated from
the reference itself (tests/golden/make_golden.py).  Each function cites the
reference lines it restates.

Parity definition for codes: numpy's float32 arctan2 is a SIMD approximation,
so a GPU (correctly rounded) angle code may differ from this oracle only for
points within ~1e-6 rad of a bin edge.  ``classify_angle_mismatch`` decides
whether a mismatch is such an admissible tie.
"""

from __future__ import annotations

import math

import numpy as np

HALF_SPLIT, ADJACENT = 1, 0
PI = np.pi
TWO_PI = 2.0 * np.pi  # tensor_core.py:22 (a Python float: arrays stay float32)


# --------------------------------------------------------------- layout


def split_xy(mat: np.ndarray, layout: int):
    """Component views, tensor_core.py:53-69."""
    d = mat.shape[-1]
    if layout == ADJACENT:
        return mat[..., 0::2], mat[..., 1::2]
    return mat[..., : d // 2], mat[..., d // 2 :]


def join_xy(x: np.ndarray, y: np.ndarray, layout: int) -> np.ndarray:
    """tensor_core.py:72-84."""
    out = np.empty(x.shape[:-1] + (2 * x.shape[-1],), dtype=np.result_type(x, y))
    if layout == ADJACENT:
        out[..., 0::2] = x
        out[..., 1::2] = y
    else:
        out[..., : x.shape[-1]] = x
        out[..., x.shape[-1] :] = y
    return out


# ------------------------------------------------------------------ HP-1


def polar(x: np.ndarray, y: np.ndarray):
    """to_polar, polar_codec.py:200-209: hypot and atan2 shifted into [0, 2pi)."""
    return np.hypot(x, y), np.mod(np.arctan2(y, x) + PI, TWO_PI)


def angle_code(theta: np.ndarray, m: int) -> np.ndarray:
    """quantize_angle, polar_codec.py:212-221 (rint half-even, wrap mod 2^m)."""
    hl = 1 << (m - 1)
    k = np.rint(np.asarray(theta) * (hl / PI)).astype(np.int64)
    return (k % (2 * hl)).astype(np.uint8)


def grid(m: int) -> np.ndarray:
    """angle_grid, polar_codec.py:224-233 (float64, includes the -pi shift)."""
    hl = 1 << (m - 1)
    return PI * np.arange(2 * hl, dtype=np.float64) / hl - PI


def scales_fp16(keys: np.ndarray, n: int, layout: int) -> np.ndarray:
    """compute_radius_scales, polar_codec.py:236-251 -> ChannelScales fp16 (:77)."""
    mat = np.asarray(keys, dtype=np.float32)
    if mat.shape[0] == 0:
        raise ValueError("cannot compute scales from an empty tensor")
    x, y = split_xy(mat, layout)
    r, _ = polar(x, y)
    top = r.max(axis=0).astype(np.float32)
    s16 = np.asarray(top / ((1 << n) - 1), dtype=np.float16)
    if s16.size and (np.any(s16 < 0) or not np.all(np.isfinite(s16.astype(np.float32)))):
        raise ValueError("scales must be finite and non-negative")
    return s16


def radius_code(r: np.ndarray, s32: np.ndarray, n: int):
    """_quantize_radius_counted, polar_codec.py:267-278."""
    top = (1 << n) - 1
    with np.errstate(divide="ignore", invalid="ignore"):
        raw = np.rint(r / s32)
    raw = np.where(s32 == 0.0, 0.0, raw)
    return np.clip(raw, 0, top).astype(np.uint8), int(np.count_nonzero(raw > top))


def encode_block(keys: np.ndarray, s16: np.ndarray, m: int, n: int, layout: int):
    """quantize_subvectors, polar_codec.py:281-302 (canonical forms included).

    Returns (angle codes, radius codes, clamp count), uint8 (T, d/2)."""
    mat = np.asarray(keys, dtype=np.float32)
    x, y = split_xy(mat, layout)
    r, theta = polar(x, y)
    a = angle_code(theta, m)
    s32 = s16.astype(np.float32)
    rc, clamped = radius_code(r, s32, n)
    a = np.where(rc == 0, np.uint8(1 << (m - 1)), a)
    dead = s32 == 0.0
    if np.any(dead):
        a = np.where(dead, np.uint8(0), a)
        rc = np.where(dead, np.uint8(0), rc)
    return a.astype(np.uint8), rc.astype(np.uint8), clamped


def pack(codes: np.ndarray, bits: int) -> bytes:
    """pack_stream, polar_codec.py:98-110 (LSB-first, token-major)."""
    flat = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1)
    if flat.size == 0:
        return b""
    planes = (flat[:, None] >> np.arange(bits, dtype=np.uint8)) & 1
    return np.packbits(planes.reshape(-1), bitorder="little").tobytes()


def unpack(stream: bytes, bits: int, count: int) -> np.ndarray:
    """unpack_stream, polar_codec.py:112-123."""
    if count == 0:
        return np.zeros(0, dtype=np.uint8)
    raw = np.frombuffer(stream, dtype=np.uint8)
    b = np.unpackbits(raw, count=count * bits, bitorder="little").reshape(count, bits).astype(np.uint16)
    return (b << np.arange(bits, dtype=np.uint16)).sum(axis=1).astype(np.uint8)


def dequantize(angle: np.ndarray, radius: np.ndarray, s16: np.ndarray, m: int, layout: int) -> np.ndarray:
    """dequantize_subvectors + merge_pairs, polar_codec.py:305-316, tensor_core.py:72-84."""
    g = grid(m)
    c, s = np.cos(g).astype(np.float32), np.sin(g).astype(np.float32)
    rhat = radius.astype(np.float32) * s16.astype(np.float32)
    return join_xy(rhat * c[angle], rhat * s[angle], layout)


# ------------------------------------------------------------------ HP-2


def angle_unit_table(m: int):
    """build_angle_table, lut_decode.py:63-74."""
    g = grid(m)
    return np.cos(g).astype(np.float32), np.sin(g).astype(np.float32)


def query_table(q: np.ndarray, m: int, layout: int) -> np.ndarray:
    """build_query_lut, lut_decode.py:86-104: (d/2, 2^m) float32."""
    c, s = angle_unit_table(m)
    qv = np.asarray(q, dtype=np.float32).reshape(-1)
    qx, qy = split_xy(qv, layout)
    return (qx[:, None] * c[None, :] + qy[:, None] * s[None, :]).astype(np.float32)


def radius_levels(s16: np.ndarray, n: int) -> np.ndarray:
    """PackedKVCache.radius_table, kv_cache.py:228-237."""
    return s16.astype(np.float32)[:, None] * np.arange(1 << n, dtype=np.float32)[None, :]


def lut_scores(q: np.ndarray, angle: np.ndarray, radius: np.ndarray, s16: np.ndarray, m: int, n: int,
               layout: int, residual: np.ndarray | None = None) -> np.ndarray:
    """qk_scores, lut_decode.py:119-154, with _residual_scores :107-116.

    Channel-major float32 accumulation, quantized tokens then residual."""
    qv = np.asarray(q, dtype=np.float32).reshape(-1)
    table = query_table(qv, m, layout)
    rtab = radius_levels(s16, n)
    acc = np.zeros(angle.shape[0], dtype=np.float32)
    for j in range(angle.shape[1]):
        acc += table[j, angle[:, j]] * rtab[j, radius[:, j]]
    if residual is None or residual.shape[0] == 0:
        tail = np.zeros(0, dtype=np.float32)
    else:
        tail = (residual.astype(np.float32) @ qv).astype(np.float32)
    return np.concatenate([acc, tail])


def softmax64(scores: np.ndarray, temperature: float) -> np.ndarray:
    """attention_weights, lut_decode.py:189-206 (float64)."""
    z = np.asarray(scores, dtype=np.float64).reshape(-1) * float(temperature)
    if z.size == 0:
        raise ValueError("cannot take attention weights of an empty score vector")
    z -= z.max()
    w = np.exp(z)
    return w / w.sum()


def attend(weights: np.ndarray, values: np.ndarray) -> np.ndarray:
    """softmax . V -- not in the reference; restated over
    PackedKVCache.values() (kv_cache.py:247-259) in float64."""
    return weights @ np.asarray(values, dtype=np.float64)


def quantize_values(values: np.ndarray, bits: int):
    """quantize_uniform(values, bits, PER_TOKEN), baseline_quant.py:58-66, 69-110:
    per row zp = min, scale = fl32(fl32(max - zp) / (2^b - 1)),
    code = clip(rint(fl32(fl32(v - zp) / scale)), 0, 2^b - 1) (scale 0 -> 0).
    Returns (codes uint8 [T, d], zero_point [T], scale [T]) in float32."""
    v = np.asarray(values, dtype=np.float32)
    top = (1 << bits) - 1
    zp = v.min(axis=1, keepdims=True)
    scale = (v.max(axis=1, keepdims=True) - zp) / np.float32(top)
    with np.errstate(divide="ignore", invalid="ignore"):
        raw = np.rint((v - zp) / scale)
    raw = np.where(scale == 0.0, np.float32(0.0), raw)
    codes = np.clip(raw, 0, top).astype(np.uint8)
    return codes, zp[:, 0].astype(np.float32), scale[:, 0].astype(np.float32)


def dequantize_values(codes: np.ndarray, zero_point: np.ndarray, scale: np.ndarray) -> np.ndarray:
    """dequantize_uniform PER_TOKEN, baseline_quant.py:143-167: fl32(fl32(code * scale) + zp)."""
    c = np.asarray(codes).astype(np.float32)
    return (c * np.asarray(scale, np.float32)[:, None] + np.asarray(zero_point, np.float32)[:, None]).astype(
        np.float32)


# ------------------------------------------------------------ the cache


class OracleCache:
    """PackedKVCache state machine, kv_cache.py:85-209 (values kept float32)."""

    def __init__(self, m: int, n: int, layout: int, residual_len: int):
        self.m, self.n, self.layout, self.s = m, n, layout, residual_len
        self.s16 = None
        self.angle = []
        self.radius = []
        self.residual = []
        self.values = []
        self.clamps = 0

    def prefill(self, keys: np.ndarray, values: np.ndarray | None = None) -> None:
        """kv_cache.py:152-177."""
        mat = np.asarray(keys, dtype=np.float32)
        if mat.size and not np.all(np.isfinite(mat)):
            raise ValueError("keys contain non-finite values")
        self.dim = mat.shape[1]
        self.s16 = scales_fp16(mat, self.n, self.layout)
        cut = max(0, mat.shape[0] - self.s)
        if cut:
            self._encode(mat[:cut])
        self.residual = [np.array(r, dtype=np.float32) for r in mat[cut:]]
        self._values(mat.shape[0], values)

    def append(self, key: np.ndarray, value: np.ndarray | None = None) -> None:
        """kv_cache.py:179-189."""
        self.residual.append(np.asarray(key, dtype=np.float32).reshape(-1).copy())
        while len(self.residual) > self.s:
            self._encode(self.residual.pop(0)[None, :])
        self._values(1, None if value is None else np.asarray(value)[None, :])

    def _encode(self, block: np.ndarray) -> None:
        a, r, c = encode_block(block, self.s16, self.m, self.n, self.layout)
        self.clamps += c
        self.angle.append(a)
        self.radius.append(r)

    def _values(self, count: int, values) -> None:
        v = np.zeros((count, self.dim), np.float32) if values is None else np.asarray(values, np.float32)
        self.values.append(v.copy())

    def codes(self):
        half = self.dim // 2
        if not self.angle:
            e = np.zeros((0, half), np.uint8)
            return e, e
        return np.concatenate(self.angle), np.concatenate(self.radius)

    def residual_keys(self) -> np.ndarray:
        if not self.residual:
            return np.zeros((0, self.dim), np.float32)
        return np.stack(self.residual)

    def all_values(self) -> np.ndarray:
        return np.concatenate(self.values)

    def scores(self, q: np.ndarray) -> np.ndarray:
        a, r = self.codes()
        return lut_scores(q, a, r, self.s16, self.m, self.n, self.layout, self.residual_keys())

    def attention(self, q: np.ndarray, temperature: float) -> np.ndarray:
        return attend(softmax64(self.scores(q), temperature), self.all_values())


# ------------------------------------------------------- synthetic inputs


def synthetic_keys(tokens: int, dim: int, seed: int, layout: int = HALF_SPLIT, log_mean: float = 0.0,
                   log_std: float = 0.5, outliers=(), boost: float = 3.0) -> np.ndarray:
    """gen_synthetic_keys, tensor_core.py:226-241 (same PCG64 draws, same order)."""
    half = dim // 2
    mean = np.full(half, float(log_mean))
    std = np.full(half, float(log_std))
    if outliers:
        mean[np.array(sorted(outliers), dtype=np.intp)] += boost
    rng = np.random.default_rng(seed)
    rad = rng.lognormal(mean=mean, sigma=std, size=(tokens, half))
    ang = rng.uniform(0.0, TWO_PI, size=(tokens, half))
    x = (rad * np.cos(ang)).astype(np.float32)
    y = (rad * np.sin(ang)).astype(np.float32)
    return np.ascontiguousarray(join_xy(x, y, layout))


# ------------------------------------------------------------ tie rules


def edge_distance(x: np.ndarray, y: np.ndarray, m: int) -> np.ndarray:
    """Distance (rad) of the float64 angle atan2(y,x)+pi to the nearest bin edge
    pi*(j + 1/2)/2^(m-1)."""
    t = np.arctan2(np.asarray(y, np.float64), np.asarray(x, np.float64)) + math.pi
    step = math.pi / (1 << (m - 1))
    u = t / step
    return np.abs(u - np.floor(u) - 0.5) * step


def classify_angle_mismatch(x, y, m: int, bound: float = 4 * float(np.spacing(np.float32(np.pi)))) -> np.ndarray:
    """True where a mismatching angle code is an admissible tie: within ``bound``
    (default 4 ulp(pi_f32) ~ 9.5e-7 rad) of a bin edge."""
    return edge_distance(x, y, m) <= bound


def radius_tie(x, y, s32, bound: float = 2.0**-20) -> np.ndarray:
    """Admissible radius-code mismatch: r64/s32 within 2^-20 relative of a half-integer."""
    r = np.hypot(np.asarray(x, np.float64), np.asarray(y, np.float64))
    q = r / np.asarray(s32, np.float64)
    return np.abs(q - np.floor(q) - 0.5) <= bound * np.maximum(q, 1.0)
