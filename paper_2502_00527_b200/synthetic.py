"""Synthetic post-RoPE keys, values and queries.

``gen_synthetic_keys`` is the reference generator itself (tensor_core.py:226-241):
numpy's PCG64 stream seeded with ``cfg.seed``, per sub-channel lognormal radius,
uniform angle, outlier channels with a boosted log-mean -- the same config and
seed give the same bytes as ``polarquant.gen_synthetic_keys``.  It is input
generation, not part of the hot path, and runs on the host like the
reference's.

``synthetic_keys_device`` / ``normal_device`` draw the same distribution with a
counter-based Philox stream on the GPU, so the benchmark can materialize tens
of GB of cache without a host round trip.  That stream is not PCG64: the
benchmark's parity leg copies the sampled units' device keys to the host and
checks them against the oracle there.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import DTYPE_CODE, layout_code, ptr, require_cuda, stream_ptr
from .core import TWO_PI, KeyTensor, PairingLayout, merge_pairs


@dataclass(frozen=True)
class SyntheticConfig:
    """Generator parameters (tensor_core.py:188-223): radius_log_mean /
    radius_log_std are scalars or (d/2,) arrays (stored broadcast to (d/2,))."""

    num_tokens: int
    dim: int
    radius_log_mean: np.ndarray = field(default=0.0)
    radius_log_std: np.ndarray = field(default=0.5)
    outlier_channels: frozenset = field(default_factory=frozenset)
    outlier_log_boost: float = 3.0
    seed: int = 0
    layout: PairingLayout = PairingLayout.HALF_SPLIT

    def __post_init__(self) -> None:
        if self.num_tokens < 0:
            raise ValueError(f"num_tokens must be >= 0, got {self.num_tokens}")
        if self.dim < 2 or self.dim % 2:
            raise ValueError(f"dim must be even and >= 2, got {self.dim}")
        half = self.dim // 2
        mean = np.broadcast_to(np.asarray(self.radius_log_mean, dtype=np.float64), (half,)).copy()
        std = np.broadcast_to(np.asarray(self.radius_log_std, dtype=np.float64), (half,)).copy()
        if np.any(std < 0):
            raise ValueError("radius_log_std must be non-negative")
        chans = frozenset(int(c) for c in self.outlier_channels)
        if any(c < 0 or c >= half for c in chans):
            raise ValueError(f"outlier channel index out of range [0, {half})")
        object.__setattr__(self, "radius_log_mean", mean)
        object.__setattr__(self, "radius_log_std", std)
        object.__setattr__(self, "outlier_channels", chans)

    def _device_params(self) -> tuple[float, float, int]:
        """(mean, std, outlier mask) for the Philox generator, which takes one
        log-mean / log-std for all channels and outliers among channels < 64."""
        mean, std = self.radius_log_mean, self.radius_log_std
        if np.ptp(mean) != 0 or np.ptp(std) != 0:
            raise ValueError("the device generator takes a scalar radius_log_mean / radius_log_std")
        if any(c >= 64 for c in self.outlier_channels):
            raise ValueError("the device generator supports outlier channels < 64")
        mask = 0
        for c in self.outlier_channels:
            mask |= 1 << c
        return float(mean[0]), float(std[0]), mask


def synthetic_keys_device(cfg: SyntheticConfig, n_units: int = 1, *, dtype: torch.dtype = torch.bfloat16,
                          device=None, seed: int | None = None) -> torch.Tensor:
    """[n_units, T, d] keys on the device; unit u is Philox stream (seed, u)."""
    dev = require_cuda(device)
    mean, std, mask = cfg._device_params()
    out = torch.empty((n_units, cfg.num_tokens, cfg.dim), dtype=dtype, device=dev)
    _lib.call(
        "pqb_synthetic_keys", int(cfg.seed if seed is None else seed) & (2**64 - 1), n_units, cfg.num_tokens,
        cfg.dim, layout_code(cfg.layout), mean, std, mask, float(cfg.outlier_log_boost), ptr(out),
        DTYPE_CODE[dtype], stream_ptr(dev),
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
    """Deterministic synthetic post-rotation keys (tensor_core.py:226-241): the
    reference's PCG64 draws in the reference's order, so equal configs give
    equal bytes in both packages."""
    half = cfg.dim // 2
    mean = cfg.radius_log_mean.copy()
    if cfg.outlier_channels:
        idx = np.fromiter(sorted(cfg.outlier_channels), dtype=np.intp)
        mean[idx] += cfg.outlier_log_boost
    rng = np.random.default_rng(cfg.seed)
    radius = rng.lognormal(mean=mean, sigma=cfg.radius_log_std, size=(cfg.num_tokens, half))
    theta = rng.uniform(0.0, TWO_PI, size=(cfg.num_tokens, half))
    x = (radius * np.cos(theta)).astype(np.float32)
    y = (radius * np.sin(theta)).astype(np.float32)
    return KeyTensor(merge_pairs(x, y, cfg.layout), layout=cfg.layout)
