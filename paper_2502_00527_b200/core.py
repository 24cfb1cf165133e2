"""Value types of the PolarQuant API, mirrored from the reference so callers can
switch packages without code changes.

  PairingLayout, split_pairs, merge_pairs, KeyTensor   tensor_core.py:41-117
  FormatError family                                  tensor_core.py:25-38
  QuantConfig, ChannelScales                          polar_codec.py:45-90
  stream_bytes, PolarCodes                            polar_codec.py:93-197
  BitReport, CacheSnapshot, OpCounter, AngleTable,
  QueryLUT                                            kv_cache.py:43-82, lut_decode.py:27-83

These are plain host containers (shapes, dtypes, validation).  Every arithmetic
step of the hot path -- scales, quantization, packing, unpacking, tables,
scores, softmax, attention -- runs in libpqb200.so on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

TWO_PI = 2.0 * np.pi
_MAX_BITS = 8


class FormatError(ValueError):
    """A binary container could not be decoded."""


class BadMagicError(FormatError):
    """The file does not start with the expected magic bytes."""


class TruncatedFileError(FormatError):
    """The file ends before the declared header or payload is complete."""


class PayloadMismatchError(FormatError):
    """The payload size disagrees with the dimensions declared in the header."""


class PairingLayout(Enum):
    """ADJACENT pairs dims (2j, 2j+1); HALF_SPLIT pairs (j, j + d/2) (the default)."""

    ADJACENT = 0
    HALF_SPLIT = 1


def split_pairs(matrix, layout: PairingLayout):
    """(x, y) component views of every 2-D sub-vector (tensor_core.py:53-69)."""
    d = matrix.shape[-1]
    if d < 2 or d % 2:
        raise ValueError(f"vector dimension must be even and >= 2, got {d}")
    if layout is PairingLayout.ADJACENT:
        return matrix[..., 0::2], matrix[..., 1::2]
    return matrix[..., : d // 2], matrix[..., d // 2 :]


def merge_pairs(x: np.ndarray, y: np.ndarray, layout: PairingLayout) -> np.ndarray:
    """Inverse of split_pairs (tensor_core.py:72-84)."""
    if x.shape != y.shape:
        raise ValueError(f"component shapes differ: {x.shape} vs {y.shape}")
    half = x.shape[-1]
    out = np.empty(x.shape[:-1] + (2 * half,), dtype=np.result_type(x, y))
    if layout is PairingLayout.ADJACENT:
        out[..., 0::2], out[..., 1::2] = x, y
    else:
        out[..., :half], out[..., half:] = x, y
    return out


@dataclass(frozen=True)
class KeyTensor:
    """(tokens, dim) float32 block with a pairing convention (tensor_core.py:87-117)."""

    data: np.ndarray
    layout: PairingLayout = PairingLayout.HALF_SPLIT

    def __post_init__(self) -> None:
        arr = np.ascontiguousarray(np.asarray(self.data, dtype=np.float32))
        if arr.ndim != 2:
            raise ValueError(f"key tensor must be 2-D, got shape {arr.shape}")
        if arr.shape[1] < 2 or arr.shape[1] % 2:
            raise ValueError(f"key dimension must be even and >= 2, got {arr.shape[1]}")
        object.__setattr__(self, "data", arr)

    @property
    def num_tokens(self) -> int:
        return self.data.shape[0]

    @property
    def dim(self) -> int:
        return self.data.shape[1]

    def subvectors(self):
        return split_pairs(self.data, self.layout)


def _check_bits(bits: int, what: str) -> None:
    if not 1 <= bits <= _MAX_BITS:
        raise ValueError(f"{what} must be in [1, {_MAX_BITS}], got {bits}")


@dataclass(frozen=True)
class QuantConfig:
    """Bit widths and pairing convention (polar_codec.py:45-63)."""

    angle_bits: int = 4
    radius_bits: int = 4
    layout: PairingLayout = PairingLayout.HALF_SPLIT

    def __post_init__(self) -> None:
        _check_bits(self.angle_bits, "angle_bits")
        _check_bits(self.radius_bits, "radius_bits")

    @property
    def angle_levels(self) -> int:
        return 1 << self.angle_bits

    @property
    def radius_levels(self) -> int:
        return 1 << self.radius_bits


@dataclass(frozen=True)
class ChannelScales:
    """Per-sub-channel radius scales stored at float16 (polar_codec.py:66-90)."""

    values: np.ndarray

    def __post_init__(self) -> None:
        arr = np.asarray(self.values, dtype=np.float16)
        if arr.ndim != 1:
            raise ValueError(f"scales must be 1-D, got shape {arr.shape}")
        if arr.size and (np.any(arr < 0) or not np.all(np.isfinite(arr.astype(np.float32)))):
            raise ValueError("scales must be finite and non-negative")
        object.__setattr__(self, "values", arr)

    @property
    def num_channels(self) -> int:
        return self.values.shape[0]

    def as_compute(self) -> np.ndarray:
        return self.values.astype(np.float32)


def stream_bytes(count: int, bits: int) -> int:
    """Packed byte length of ``count`` codes at ``bits`` bits (polar_codec.py:93-95)."""
    return (count * bits + 7) // 8


@dataclass(frozen=True)
class PolarCodes:
    """Bit-packed angle and radius streams (polar_codec.py:126-197).

    The byte format is the reference's; angle_codes()/radius_codes() unpack on
    the GPU (pqb_unpack_codes).
    """

    num_tokens: int
    dim: int
    angle_bits: int
    radius_bits: int
    layout: PairingLayout
    angle_stream: bytes
    radius_stream: bytes

    def __post_init__(self) -> None:
        if self.num_tokens < 0:
            raise ValueError(f"num_tokens must be >= 0, got {self.num_tokens}")
        if self.dim < 2 or self.dim % 2:
            raise ValueError(f"dim must be even and >= 2, got {self.dim}")
        _check_bits(self.angle_bits, "angle_bits")
        _check_bits(self.radius_bits, "radius_bits")
        count = self.num_tokens * (self.dim // 2)
        for name, stream, bits in (
            ("angle", self.angle_stream, self.angle_bits),
            ("radius", self.radius_stream, self.radius_bits),
        ):
            if len(stream) != stream_bytes(count, bits):
                raise ValueError(f"{name} stream has {len(stream)} bytes, expected {stream_bytes(count, bits)}")

    @classmethod
    def from_arrays(cls, angle, radius, cfg: QuantConfig, dim: int | None = None) -> "PolarCodes":
        """Pack (T, d/2) code arrays on the GPU (pack_stream semantics)."""
        from .codec import pack_code_arrays

        angle = np.asarray(angle)
        radius = np.asarray(radius)
        if angle.shape != radius.shape or angle.ndim != 2:
            raise ValueError(f"code arrays must share a (T, d/2) shape, got {angle.shape} and {radius.shape}")
        half = angle.shape[1]
        dim = 2 * half if dim is None else dim
        if dim != 2 * half:
            raise ValueError(f"dim {dim} does not match {half} sub-channels")
        a_stream, r_stream = pack_code_arrays(angle, radius, cfg)
        return cls(angle.shape[0], dim, cfg.angle_bits, cfg.radius_bits, cfg.layout, a_stream, r_stream)

    def angle_codes(self) -> np.ndarray:
        from .codec import unpack_streams

        return unpack_streams(self)[0]

    def radius_codes(self) -> np.ndarray:
        from .codec import unpack_streams

        return unpack_streams(self)[1]

    def config(self) -> QuantConfig:
        return QuantConfig(self.angle_bits, self.radius_bits, self.layout)


@dataclass(frozen=True)
class BitReport:
    """Key-cache storage accounting in bits (kv_cache.py:43-71)."""

    payload_bits: int
    param_bits: int
    residual_bits: int
    avg_bits_per_element: float
    payload_bits_per_element: float
    num_tokens: int
    quantized_tokens: int
    residual_tokens: int

    @property
    def total_bits(self) -> int:
        return self.payload_bits + self.param_bits + self.residual_bits

    def as_dict(self) -> dict:
        return {
            "payload_bits": self.payload_bits,
            "param_bits": self.param_bits,
            "residual_bits": self.residual_bits,
            "total_bits": self.total_bits,
            "avg_bits_per_element": self.avg_bits_per_element,
            "payload_bits_per_element": self.payload_bits_per_element,
            "num_tokens": self.num_tokens,
            "quantized_tokens": self.quantized_tokens,
            "residual_tokens": self.residual_tokens,
        }


@dataclass(frozen=True)
class CacheSnapshot:
    """Immutable cache view (kv_cache.py:74-82)."""

    codes: PolarCodes
    scales: ChannelScales
    residual_keys: np.ndarray
    residual_len: int
    clamp_events: int


@dataclass
class OpCounter:
    """Arithmetic tally (lut_decode.py:27-47).  The GPU kernels execute the
    reference's operation sequence; score calls add the counts that sequence
    performs (the same closed forms the reference's instrumented loop yields)."""

    multiplies: int = 0
    additions: int = 0
    lookups: int = 0

    def reset(self) -> None:
        self.multiplies = self.additions = self.lookups = 0

    def as_dict(self) -> dict:
        return {"multiplies": self.multiplies, "additions": self.additions, "lookups": self.lookups}


@dataclass(frozen=True)
class AngleTable:
    """Unit vectors of every decoded grid angle, float32 (lut_decode.py:50-60)."""

    cos: np.ndarray
    sin: np.ndarray
    angle_bits: int

    def unit_vectors(self) -> np.ndarray:
        return np.stack([self.cos, self.sin], axis=1)


@dataclass(frozen=True)
class QueryLUT:
    """Per-sub-channel partial dot products of one query, (d/2, 2^m) (lut_decode.py:77-83)."""

    partial: np.ndarray
    angle_bits: int
    layout: PairingLayout
