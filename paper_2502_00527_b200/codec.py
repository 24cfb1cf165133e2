"""HP-1 public API: compute_radius_scales / encode_keys / decode_keys on the GPU.

Same names, argument meanings and error behaviour as the reference
(polar_codec.py:236-251, 319-364); the work is done by K1 (pqb_radius_scales)
and K2 (pqb_encode) in libpqb200.so.  Batched device entry points
(``radius_scales_device``, ``encode_device``) serve the paged cache and the
benchmark without host round trips.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._device import (
    ContigStore,
    as_device_matrix,
    dtype_code,
    layout_code,
    new_flags,
    ptr,
    raise_on_flags,
    require_cuda,
    stream_ptr,
)
from .core import ChannelScales, KeyTensor, PolarCodes, QuantConfig, _check_bits, merge_pairs, stream_bytes


def radius_scales_device(keys: torch.Tensor, cfg: QuantConfig, flags: torch.Tensor | None = None,
                         workspace: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """K1 over a device tensor [U, T, d] (or [T, d]); returns fp16 scales [U, d/2].

    Asynchronous: non-finite inputs / fp16 overflow are reported in ``flags``."""
    k3 = keys if keys.dim() == 3 else keys.unsqueeze(0)
    if k3.stride(-1) != 1:
        k3 = k3.contiguous()
    U, T, d = k3.shape
    if d < 2 or d % 2:
        raise ValueError(f"vector dimension must be even and >= 2, got {d}")
    half = d // 2
    dev = k3.device
    if out is None:
        out = torch.empty((U, half), dtype=torch.float16, device=dev)
    ws = workspace if workspace is not None else torch.empty(U * half, dtype=torch.int64, device=dev)
    flags = flags if flags is not None else new_flags(dev)
    _lib.call(
        "pqb_radius_scales", ptr(k3), dtype_code(k3), U, T, d, k3.stride(0), k3.stride(1),
        layout_code(cfg.layout), cfg.radius_bits, ptr(ws), ptr(out), ptr(flags), stream_ptr(dev),
    )
    return out


def encode_device(keys: torch.Tensor, scales: torch.Tensor, cfg: QuantConfig, store_ref, *, tok_offset=None,
                  tok_offset_const: int = 0, clamp_counts: torch.Tensor | None = None,
                  flags: torch.Tensor | None = None) -> None:
    """K2 over a device tensor [U, T, d] into a paged store (ctypes pointer to PqbStore)."""
    k3 = keys if keys.dim() == 3 else keys.unsqueeze(0)
    if k3.stride(-1) != 1:
        k3 = k3.contiguous()
    U, T, d = k3.shape
    dev = k3.device
    flags = flags if flags is not None else new_flags(dev)
    sc = scales.contiguous()
    _lib.call(
        "pqb_encode", ptr(k3), dtype_code(k3), U, T, d, k3.stride(0), k3.stride(1), layout_code(cfg.layout),
        cfg.angle_bits, cfg.radius_bits, ptr(sc), store_ref, ptr(tok_offset), tok_offset_const,
        ptr(clamp_counts), ptr(flags), stream_ptr(dev),
    )


def _matrix(keys) -> torch.Tensor:
    dev = require_cuda()
    return as_device_matrix(keys, dev)


def compute_radius_scales(keys: KeyTensor | np.ndarray, cfg: QuantConfig) -> ChannelScales:
    """Per-sub-channel scales: max radius over tokens / top radius code.

    polar_codec.py:236-251.  Raises ValueError on an empty tensor."""
    m = _matrix(keys)
    if m.dim() != 2:
        raise ValueError(f"keys must be 2-D, got shape {tuple(m.shape)}")
    if m.shape[0] == 0:
        raise ValueError("cannot compute scales from an empty tensor")
    flags = new_flags(m.device)
    s16 = radius_scales_device(m, cfg, flags)
    raise_on_flags(flags, "compute_radius_scales")
    return ChannelScales(s16[0].cpu().numpy())


def _scales_device(scales: ChannelScales, device: torch.device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(scales.values)).to(device).view(torch.float16)


def encode_keys(keys: KeyTensor | np.ndarray, scales: ChannelScales, cfg: QuantConfig) -> PolarCodes:
    """Quantize a key block against fixed channel scales (polar_codec.py:319-344)."""
    m = _matrix(keys)
    if m.dim() != 2:
        raise ValueError(f"keys must be 2-D, got shape {tuple(m.shape)}")
    T, d = m.shape
    if scales.num_channels != d // 2:
        raise ValueError(f"{scales.num_channels} scales for {d} dims (need d/2)")
    if d < 2 or d % 2:
        raise ValueError(f"vector dimension must be even and >= 2, got {d}")
    store = ContigStore(1, T, d, cfg.angle_bits, cfg.radius_bits, m.device)
    flags = new_flags(m.device)
    if T:
        encode_device(m, _scales_device(scales, m.device), cfg, store.ref(), flags=flags)
        raise_on_flags(flags, "encode_keys")
    count = T * (d // 2)
    return PolarCodes(
        num_tokens=T,
        dim=d,
        angle_bits=cfg.angle_bits,
        radius_bits=cfg.radius_bits,
        layout=cfg.layout,
        angle_stream=store.angle_bytes(0, stream_bytes(count, cfg.angle_bits)),
        radius_stream=store.radius_bytes(0, stream_bytes(count, cfg.radius_bits)),
    )


def _upload_codes(codes: PolarCodes, device: torch.device) -> ContigStore:
    """Place a PolarCodes' two streams into a one-page device store."""
    store = ContigStore(1, codes.num_tokens, codes.dim, codes.angle_bits, codes.radius_bits, device)
    for off, stream in ((store.angle_off, codes.angle_stream), (store.radius_off, codes.radius_stream)):
        if stream:
            src = torch.frombuffer(bytearray(stream), dtype=torch.uint8)
            store.pool[off : off + len(stream)].copy_(src)
    return store


def unpack_streams(codes: PolarCodes) -> tuple[np.ndarray, np.ndarray]:
    """PolarCodes.angle_codes / radius_codes (polar_codec.py:182-194) via pqb_unpack_codes."""
    dev = require_cuda()
    half = codes.dim // 2
    T = codes.num_tokens
    a = torch.empty((T, half), dtype=torch.uint8, device=dev)
    r = torch.empty((T, half), dtype=torch.uint8, device=dev)
    if T:
        store = _upload_codes(codes, dev)
        _lib.call("pqb_unpack_codes", store.ref(), 0, codes.dim, codes.angle_bits, codes.radius_bits, T,
                  ptr(a), ptr(r), stream_ptr(dev))
    return a.cpu().numpy(), r.cpu().numpy()


def pack_code_arrays(angle: np.ndarray, radius: np.ndarray, cfg: QuantConfig) -> tuple[bytes, bytes]:
    """pack_stream of both (T, d/2) arrays (polar_codec.py:98-110) via pqb_pack_codes."""
    dev = require_cuda()
    T, half = angle.shape
    d = 2 * half
    count = T * half
    if count == 0:
        return b"", b""
    store = ContigStore(1, T, d, cfg.angle_bits, cfg.radius_bits, dev)
    a = torch.from_numpy(np.ascontiguousarray(angle, dtype=np.uint8)).to(dev)
    r = torch.from_numpy(np.ascontiguousarray(radius, dtype=np.uint8)).to(dev)
    _lib.call("pqb_pack_codes", ptr(a), ptr(r), T, d, cfg.angle_bits, cfg.radius_bits, store.ref(), 0,
              stream_ptr(dev))
    return (store.angle_bytes(0, stream_bytes(count, cfg.angle_bits)),
            store.radius_bytes(0, stream_bytes(count, cfg.radius_bits)))


def dequantize_store(store_struct, scales16: torch.Tensor, cfg: QuantConfig, d: int, unit: int, tokens: int,
                     device: torch.device) -> torch.Tensor:
    """GPU dequantize_subvectors + merge_pairs for one unit -> fp32 [tokens, d]."""
    out = torch.empty((tokens, d), dtype=torch.float32, device=device)
    if tokens:
        cache = _lib.PqbCache(store=store_struct, d=d, angle_bits=cfg.angle_bits, radius_bits=cfg.radius_bits,
                              layout=layout_code(cfg.layout), scales=ptr(scales16), seq_lens=None, quant_lens=None,
                              residual=None, res_cap=0, reserved=0)
        _lib.call("pqb_dequantize", ctypes.byref(cache), unit, tokens, ptr(out), stream_ptr(device))
    return out


def decode_keys(codes: PolarCodes, scales: ChannelScales, cfg: QuantConfig | None = None) -> KeyTensor:
    """Reconstruct a float32 key block from packed codes (polar_codec.py:347-364)."""
    if cfg is not None and cfg != codes.config():
        raise ValueError(f"config {cfg} does not match codes {codes.config()}")
    if scales.num_channels != codes.dim // 2:
        raise ValueError(f"{scales.num_channels} scales for {codes.dim} dims (need d/2)")
    dev = require_cuda()
    store = _upload_codes(codes, dev)
    out = dequantize_store(store.struct, _scales_device(scales, dev), codes.config(), codes.dim, 0,
                           codes.num_tokens, dev)
    return KeyTensor(out.cpu().numpy(), layout=codes.layout)


__all__ = [
    "compute_radius_scales",
    "encode_keys",
    "decode_keys",
    "radius_scales_device",
    "encode_device",
    "unpack_streams",
    "pack_code_arrays",
    "merge_pairs",
]


# ------------------------------------------------------------------ element-wise
# The reference's array-level functions (polar_codec.py:200-278), on the GPU.
# numpy computes them in the operands' precision (NEP 50: Python floats are weak
# and take the array's dtype), so float32 arrays run the float32 kernels and
# float64 arrays / Python scalars / integers the float64 ones.  Inputs are
# broadcast on the host like numpy; 0-d inputs return numpy scalars.


def _precision(*xs) -> np.dtype:
    dt = np.result_type(*(x if isinstance(x, (int, float, np.ndarray, np.generic)) else np.asarray(x) for x in xs))
    if dt == np.float32 or dt == np.float16:  # float16: computed in float32 (numpy would round each step to fp16)
        return np.dtype(np.float32)
    return np.dtype(np.float64)


def _to_device(a: np.ndarray, dev: torch.device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _scalar_or_array(out: np.ndarray, ndim: int):
    return out[()] if ndim == 0 else out


def to_polar(x, y) -> tuple[np.ndarray, np.ndarray]:
    """(radius, angle) of Cartesian components (polar_codec.py:200-209):
    radius = hypot(x, y), angle = mod(atan2(y, x) + pi, 2 pi) in [0, 2 pi);
    the origin maps to angle pi.  float32: hypotf's exact rounding and a
    correctly rounded atan2 (numpy's SIMD arctan2 may differ by a few ulp)."""
    dev = require_cuda()
    dt = _precision(x, y)
    xb, yb = np.broadcast_arrays(np.asarray(x, dtype=dt), np.asarray(y, dtype=dt))
    n = xb.size
    xd, yd = _to_device(xb.reshape(-1), dev), _to_device(yb.reshape(-1), dev)
    tdt = torch.float32 if dt == np.float32 else torch.float64
    r = torch.empty(n, dtype=tdt, device=dev)
    t = torch.empty(n, dtype=tdt, device=dev)
    if n:
        _lib.call("pqb_to_polar", ptr(xd), ptr(yd), _lib.PQB_F32 if dt == np.float32 else _lib.PQB_F64, n, ptr(r),
                  ptr(t), stream_ptr(dev))
    shape = xb.shape
    return (_scalar_or_array(r.cpu().numpy().reshape(shape), len(shape)),
            _scalar_or_array(t.cpu().numpy().reshape(shape), len(shape)))


def quantize_angle(theta, angle_bits: int) -> np.ndarray:
    """Nearest point of the circular 2^m grid, half-even, wrapping 2 pi to 0
    (polar_codec.py:212-221)."""
    _check_bits(angle_bits, "angle_bits")
    dev = require_cuda()
    dt = _precision(theta)
    th = np.asarray(theta, dtype=dt)
    n = th.size
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    if n:
        thd = _to_device(th.reshape(-1), dev)  # held until the call is enqueued
        _lib.call("pqb_quantize_angle", ptr(thd),
                  _lib.PQB_F32 if dt == np.float32 else _lib.PQB_F64, n, angle_bits, ptr(out), stream_ptr(dev))
    return _scalar_or_array(out.cpu().numpy().reshape(th.shape), th.ndim)


def angle_grid(angle_bits: int) -> np.ndarray:
    """Decoded angle of every code, float64, in [-pi, pi) (polar_codec.py:224-233)."""
    _check_bits(angle_bits, "angle_bits")
    dev = require_cuda()
    out = torch.empty(1 << angle_bits, dtype=torch.float64, device=dev)
    _lib.call("pqb_angle_grid", angle_bits, ptr(out), stream_ptr(dev))
    return out.cpu().numpy()


def quantize_radius_counted(radius, scale, radius_bits: int) -> tuple[np.ndarray, int]:
    """_quantize_radius_counted (polar_codec.py:267-278): codes plus the number
    of entries clamped from above."""
    _check_bits(radius_bits, "radius_bits")
    dev = require_cuda()
    r = np.asarray(radius)
    s32 = np.asarray(scale).astype(np.float32)
    dt = _precision(r, s32)
    rb, sb = np.broadcast_arrays(r.astype(dt, copy=False), s32)
    n = rb.size
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    clamped = torch.zeros(1, dtype=torch.int64, device=dev)
    if n:
        rd, sd = _to_device(rb.reshape(-1), dev), _to_device(sb.reshape(-1), dev)  # both alive across the call
        _lib.call("pqb_quantize_radius", ptr(rd),
                  _lib.PQB_F32 if dt == np.float32 else _lib.PQB_F64, ptr(sd), n,
                  radius_bits, ptr(out), ptr(clamped), stream_ptr(dev))
    return _scalar_or_array(out.cpu().numpy().reshape(rb.shape), rb.ndim), int(clamped.item())


def quantize_radius(radius, scale, radius_bits: int) -> np.ndarray:
    """Round radii to code * scale points, clamping to the code range; zero
    scales force code 0; broadcasting applies (polar_codec.py:254-264)."""
    return quantize_radius_counted(radius, scale, radius_bits)[0]


__all__ += ["to_polar", "quantize_angle", "angle_grid", "quantize_radius"]
