"""Seeded on-device synthetic post-RoPE keys, values and queries.

Same distribution as the reference generator (tensor_core.py:188-241: per
sub-channel lognormal radius, uniform angle, optional outlier channels with a
boosted log-mean), drawn with a counter-based Philox stream on the GPU so the
benchmark can materialize 10s of GB of cache without a host round trip.  The
stream is not numpy's PCG64: parity tests that need the reference's exact bytes
generate them with the oracle instead.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import DTYPE_CODE, layout_code, ptr, require_cuda, stream_ptr
from .core import KeyTensor, PairingLayout


@dataclass(frozen=True)
class SyntheticConfig:
    """Generator parameters (tensor_core.py:188-223)."""

    num_tokens: int
    dim: int
    radius_log_mean: float = 0.0
    radius_log_std: float = 0.5
    outlier_channels: frozenset = field(default_factory=frozenset)
    outlier_log_boost: float = 3.0
    seed: int = 0
    layout: PairingLayout = PairingLayout.HALF_SPLIT

    def __post_init__(self) -> None:
        if self.num_tokens < 0:
            raise ValueError(f"num_tokens must be >= 0, got {self.num_tokens}")
        if self.dim < 2 or self.dim % 2:
            raise ValueError(f"dim must be even and >= 2, got {self.dim}")
        if self.radius_log_std < 0:
            raise ValueError("radius_log_std must be non-negative")
        half = self.dim // 2
        chans = frozenset(int(c) for c in self.outlier_channels)
        if any(c < 0 or c >= half for c in chans):
            raise ValueError(f"outlier channel index out of range [0, {half})")
        if any(c >= 64 for c in chans):
            raise ValueError("the device generator supports outlier channels < 64")
        object.__setattr__(self, "outlier_channels", chans)


def synthetic_keys_device(cfg: SyntheticConfig, n_units: int = 1, *, dtype: torch.dtype = torch.bfloat16,
                          device=None, seed: int | None = None) -> torch.Tensor:
    """[n_units, T, d] keys on the device; unit u is Philox stream (seed, u)."""
    dev = require_cuda(device)
    out = torch.empty((n_units, cfg.num_tokens, cfg.dim), dtype=dtype, device=dev)
    mask = 0
    for c in cfg.outlier_channels:
        mask |= 1 << c
    _lib.call(
        "pqb_synthetic_keys", int(cfg.seed if seed is None else seed) & (2**64 - 1), n_units, cfg.num_tokens,
        cfg.dim, layout_code(cfg.layout), float(cfg.radius_log_mean), float(cfg.radius_log_std), mask,
        float(cfg.outlier_log_boost), ptr(out), DTYPE_CODE[dtype], stream_ptr(dev),
    )
    return out


def normal_device(shape, seed: int, *, dtype: torch.dtype = torch.bfloat16, device=None) -> torch.Tensor:
    """Standard-normal tensor of ``shape`` from Philox stream ``seed``."""
    dev = require_cuda(device)
    out = torch.empty(shape, dtype=dtype, device=dev)
    _lib.call("pqb_synthetic_normal", int(seed) & (2**64 - 1), out.numel(), ptr(out), DTYPE_CODE[dtype],
              stream_ptr(dev))
    return out


def gen_synthetic_keys(cfg: SyntheticConfig) -> KeyTensor:
    """Host KeyTensor drawn on the device (reference name, tensor_core.py:226-241)."""
    t = synthetic_keys_device(cfg, 1, dtype=torch.float32)[0]
    return KeyTensor(np.ascontiguousarray(t.cpu().numpy()), layout=cfg.layout)
