"""Device plumbing shared by the API modules: CUDA checks, pointers, streams,
dtype codes, and small paged-store builders.  PyTorch provides allocation and
streams only; all arithmetic is in libpqb200.so."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import KeyTensor, PairingLayout

DTYPE_CODE = {torch.float32: _lib.PQB_F32, torch.bfloat16: _lib.PQB_BF16, torch.float16: _lib.PQB_F16}


def require_cuda(device: torch.device | str | int | None = None) -> torch.device:
    """The product path has no CPU implementation: fail loudly without a GPU."""
    _lib.load()
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2502_00527_b200 runs on a CUDA device (sm_100a B200); no CUDA device is visible "
            "and there is no CPU fallback"
        )
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    return dev


def stream_ptr(device: torch.device | None = None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def dtype_code(t: torch.Tensor) -> int:
    try:
        return DTYPE_CODE[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}; expected float32, bfloat16 or float16") from None


def as_device_matrix(keys, device: torch.device) -> torch.Tensor:
    """Reference input coercion (KeyTensor / np.asarray(..., float32)) onto the device.

    numpy and KeyTensor inputs become float32 exactly as the reference casts
    them; torch tensors keep their float dtype (f32/bf16/f16 are all exact in
    f32, which is what the kernels compute in)."""
    if isinstance(keys, KeyTensor):
        keys = keys.data
    if isinstance(keys, torch.Tensor):
        t = keys
        if t.dtype not in DTYPE_CODE:
            t = t.to(torch.float32)
        return t.to(device)
    arr = np.ascontiguousarray(np.asarray(keys, dtype=np.float32))
    return torch.from_numpy(arr).to(device)


def layout_code(layout: PairingLayout) -> int:
    return int(layout.value)


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


class ContigStore:
    """One page per unit holding a whole stream: the reference's contiguous
    PolarCodes layout expressed as a (trivially) paged store."""

    def __init__(self, n_units: int, tokens: int, d: int, m: int, n: int, device: torch.device,
                 value_dtype: torch.dtype | None = None):
        half = d // 2
        self.page_tokens = max(32, round_up(tokens, 32))
        self.a_bytes = self.page_tokens * half * m // 8
        self.r_bytes = self.page_tokens * half * n // 8
        self.angle_off = 0
        self.radius_off = round_up(self.a_bytes, 16)
        self.value_off = -1
        page = self.radius_off + round_up(self.r_bytes, 16)
        self.value_dtype = value_dtype
        if value_dtype is not None:
            self.value_off = page
            page += self.page_tokens * d * (4 if value_dtype == torch.float32 else 2)
        self.page_bytes = round_up(page, 16)
        self.pool = torch.zeros(n_units * self.page_bytes, dtype=torch.uint8, device=device)
        self.struct = _lib.PqbStore(
            pool=self.pool.data_ptr(),
            page_bytes=self.page_bytes,
            angle_off=self.angle_off,
            radius_off=self.radius_off,
            value_off=self.value_off,
            page_table=None,
            max_pages=1,
            page_tokens=self.page_tokens,
            value_dtype=_lib.PQB_F32 if value_dtype in (None, torch.float32) else _lib.PQB_BF16,
            reserved=0,
        )

    def ref(self):
        return ctypes.byref(self.struct)

    def angle_bytes(self, unit: int, nbytes: int) -> bytes:
        base = unit * self.page_bytes + self.angle_off
        return bytes(self.pool[base : base + nbytes].cpu().numpy().tobytes())

    def radius_bytes(self, unit: int, nbytes: int) -> bytes:
        base = unit * self.page_bytes + self.radius_off
        return bytes(self.pool[base : base + nbytes].cpu().numpy().tobytes())


def new_flags(device: torch.device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device)


def raise_on_flags(flags: torch.Tensor, what: str) -> None:
    """Synchronizing check of the device error flags (reference raises ValueError)."""
    v = int(flags.item())
    if v & _lib.PQB_FLAG_NONFINITE:
        raise ValueError(f"{what}: keys contain non-finite values")
    if v & _lib.PQB_FLAG_SCALE_OVERFLOW:
        raise ValueError(f"{what}: scales must be finite and non-negative (fp16 overflow)")
