"""HP-2 public API: LUT scoring and fused decode attention on the GPU.

Reference names and semantics (lut_decode.py:63-206):
  build_angle_table, build_query_lut, qk_scores, qk_scores_direct,
  attention_weights
plus ``decode_attention`` -- softmax(q.K * scale).V fused in one kernel
(the reference stops at the weights).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from ._device import as_device_matrix, dtype_code, layout_code, ptr, require_cuda, stream_ptr
from .cache import PackedKVCache, PolarKVCache
from .core import AngleTable, OpCounter, PairingLayout, QueryLUT, split_pairs


def build_angle_table(angle_bits: int) -> AngleTable:
    """cos/sin of every decoded grid angle, fp32 (lut_decode.py:63-74)."""
    if not 1 <= angle_bits <= 8:
        raise ValueError(f"angle_bits must be in [1, 8], got {angle_bits}")
    dev = require_cuda()
    L = 1 << angle_bits
    c = torch.empty(L, dtype=torch.float32, device=dev)
    s = torch.empty(L, dtype=torch.float32, device=dev)
    _lib.call("pqb_angle_table", angle_bits, ptr(c), ptr(s), stream_ptr(dev))
    return AngleTable(cos=c.cpu().numpy(), sin=s.cpu().numpy(), angle_bits=angle_bits)


def build_query_lut(query, table: AngleTable, layout: PairingLayout = PairingLayout.HALF_SPLIT,
                    counter: OpCounter | None = None) -> QueryLUT:
    """P[j][a] = qx_j * cos_a + qy_j * sin_a in fp32 (lut_decode.py:86-104)."""
    dev = require_cuda()
    q = as_device_matrix(np.asarray(query, dtype=np.float32).reshape(-1)
                         if not isinstance(query, torch.Tensor) else query.reshape(-1), dev).contiguous()
    d = q.shape[0]
    split_pairs(np.empty((d,)), layout)  # reference validation: even d >= 2
    m = table.angle_bits
    out = torch.empty((d // 2, 1 << m), dtype=torch.float32, device=dev)
    _lib.call("pqb_query_lut", ptr(q), dtype_code(q), 1, d, layout_code(layout), m, ptr(out), stream_ptr(dev))
    if counter is not None:
        entries = out.numel()
        counter.multiplies += 2 * entries
        counter.additions += entries
    return QueryLUT(partial=out.cpu().numpy(), angle_bits=m, layout=layout)


def _query_row(query, cache: PackedKVCache) -> torch.Tensor:
    dev = cache.device_cache.device
    q = as_device_matrix(np.asarray(query, dtype=np.float32).reshape(-1)
                         if not isinstance(query, torch.Tensor) else query.reshape(-1), dev)
    if q.shape[0] != cache.dim:
        raise ValueError(f"query dim {q.shape[0]} != cache dim {cache.dim}")
    return q


def qk_scores(query, cache: PackedKVCache, counter: OpCounter | None = None) -> np.ndarray:
    """Scores of one query against every cached token via the query LUT.

    lut_decode.py:119-154: quantized tokens first -- bit-identical to the
    reference's fp32 channel-major accumulation -- then exact fp32 dots
    against the residual window."""
    q = _query_row(query, cache)
    dc = cache.device_cache
    T = cache.num_tokens
    sc = dc.scores(q.view(1, 1, -1), max_tokens=T)[0, 0]
    if counter is not None:
        d, tq, tr = cache.dim, cache.quantized_tokens, cache.residual_tokens
        entries = (d // 2) * cache.cfg.angle_levels
        counter.multiplies += 2 * entries + tq * (d // 2) + tr * d
        counter.additions += entries + tq * (d // 2) + tr * d
        counter.lookups += 2 * tq * (d // 2)
    return sc.cpu().numpy()


def qk_scores_direct(query, cache: PackedKVCache, counter: OpCounter | None = None) -> np.ndarray:
    """Dequantize-then-dot path (lut_decode.py:157-186): one kernel
    (pqb_scores_direct) dequantizes every quantized key exactly as
    decode_quantized (bit-identical x_hat/y_hat) and dots it with the query in
    fp32, then the residual keys -- the reference's independent check of the
    LUT path (agreement within 1e-4 of the peak, test_acceptance.py:64-92)."""
    q = _query_row(query, cache).contiguous()
    dc = cache.device_cache
    T = cache.num_tokens
    out = dc.scores_direct(q, 0, T)
    if counter is not None:
        n = cache.quantized_tokens * cache.dim
        r = cache.residual_tokens * cache.dim
        counter.lookups += 3 * n // 2
        counter.multiplies += 2 * n + r
        counter.additions += n + r
    return out.cpu().numpy()


def attention_weights(scores, temperature: float) -> np.ndarray:
    """float64 softmax of temperature-scaled scores (lut_decode.py:189-206)."""
    dev = require_cuda()
    s = torch.as_tensor(np.asarray(scores, dtype=np.float32).reshape(-1)
                        if not isinstance(scores, torch.Tensor) else scores.reshape(-1).float(), device=dev)
    if s.numel() == 0:
        raise ValueError("cannot take attention weights of an empty score vector")
    out = torch.empty(s.numel(), dtype=torch.float64, device=dev)
    s = s.contiguous()
    _lib.call("pqb_softmax_f64", ptr(s), s.numel(), float(temperature), ptr(out), stream_ptr(dev))
    return out.cpu().numpy()


def decode_attention(query, cache, sm_scale: float | None = None, *, out_dtype: torch.dtype = torch.float32):
    """Fused LUT decode attention.

    * ``cache`` a PackedKVCache: query (d,) or (G, d) -> numpy (d,) / (G, d).
    * ``cache`` a PolarKVCache: device query [U, G, d] -> device [U, G, d].
    sm_scale defaults to 1/sqrt(d), the temperature cli.py:297 uses."""
    if isinstance(cache, PolarKVCache):
        return cache.decode(query, sm_scale, out_dtype=out_dtype)
    dc = cache.device_cache
    dev = dc.device
    q = as_device_matrix(np.asarray(query, dtype=np.float32) if not isinstance(query, torch.Tensor) else query, dev)
    single = q.dim() == 1
    q3 = q.reshape(1, -1, cache.dim) if q.shape[-1] == cache.dim else None
    if q3 is None:
        raise ValueError(f"query dim {q.shape[-1]} != cache dim {cache.dim}")
    scale = (1.0 / math.sqrt(cache.dim)) if sm_scale is None else sm_scale
    out = dc.decode(q3, scale, out_dtype=out_dtype, max_tokens=cache.num_tokens)[0]
    out = out.float().cpu().numpy()
    return out[0] if single else out
