"""ctypes binding of oracle/build/libpolar_oracle.so -- TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libpolar_oracle.so"
_lib = None


def build() -> Path:
    """make under an exclusive file lock (ranks of a multi-process bench may
    all ask for the checker at once; the Makefile also renames atomically)."""
    import fcntl

    (HERE / "build").mkdir(exist_ok=True)
    with open(HERE / "build" / ".lock", "w") as fh:
        fcntl.flock(fh, fcntl.LOCK_EX)
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.pqo_scales.argtypes = [vp, i64, i32, i32, i32, vp]
        L.pqo_scales.restype = i32
        L.pqo_encode.argtypes = [vp, i64, i32, i32, i32, i32, vp, vp, vp]
        L.pqo_encode.restype = i64
        L.pqo_pack.argtypes = [vp, i64, i32, vp]
        L.pqo_lut_scores.argtypes = [vp, vp, vp, i64, i32, vp, i32, i32, i32, vp]
        L.pqo_f32_to_f16.argtypes = [ctypes.c_float]
        L.pqo_f32_to_f16.restype = ctypes.c_uint16
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def scales(keys: np.ndarray, n: int, layout: int) -> np.ndarray:
    k = np.ascontiguousarray(keys, dtype=np.float32)
    T, d = k.shape
    out = np.zeros(d // 2, dtype=np.uint16)
    lib().pqo_scales(_p(k), T, d, layout, n, _p(out))
    return out.view(np.float16)


def encode(keys: np.ndarray, s16: np.ndarray, m: int, n: int, layout: int):
    k = np.ascontiguousarray(keys, dtype=np.float32)
    T, d = k.shape
    s = np.ascontiguousarray(s16, dtype=np.float16).view(np.uint16)
    a = np.zeros((T, d // 2), dtype=np.uint8)
    r = np.zeros((T, d // 2), dtype=np.uint8)
    c = lib().pqo_encode(_p(k), T, d, layout, m, n, _p(s), _p(a), _p(r))
    return a, r, int(c)


def pack(codes: np.ndarray, bits: int) -> bytes:
    c = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1)
    out = np.zeros((c.size * bits + 7) // 8, dtype=np.uint8)
    if c.size:
        lib().pqo_pack(_p(c), c.size, bits, _p(out))
    return out.tobytes()


def lut_scores(q: np.ndarray, angle: np.ndarray, radius: np.ndarray, s16: np.ndarray, m: int, n: int,
               layout: int) -> np.ndarray:
    qv = np.ascontiguousarray(q, dtype=np.float32).reshape(-1)
    a = np.ascontiguousarray(angle, dtype=np.uint8)
    r = np.ascontiguousarray(radius, dtype=np.uint8)
    s = np.ascontiguousarray(s16, dtype=np.float16).view(np.uint16)
    out = np.zeros(a.shape[0], dtype=np.float32)
    lib().pqo_lut_scores(_p(qv), _p(a), _p(r), a.shape[0], qv.size, _p(s), m, n, layout, _p(out))
    return out
