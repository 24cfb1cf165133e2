"""ctypes binding of libpqb200.so (include/pqb200.h).

The library is built in-tree by ``python -m paper_2502_00527_b200.build`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
or no CUDA device is visible, the product API raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libpqb200.so"

PQB_OK, PQB_EINVAL, PQB_ESTATE, PQB_ECUDA, PQB_EUNSUPPORTED = 0, 1, 2, 3, 4
PQB_FLAG_NONFINITE, PQB_FLAG_SCALE_OVERFLOW = 1, 2
PQB_F32, PQB_BF16, PQB_F16 = 0, 1, 2
PQB_F64 = 3  # element-wise reference API only
PQB_VQ4 = 16  # pqb_store.value_dtype: 4-bit per-token value codes
PQB_VQ2, PQB_VQ8 = 17, 18  # 2- / 8-bit per-token value codes
PQB_DECODE_FORCE_GENERIC, PQB_DECODE_NO_COMBINE, PQB_DECODE_DQ, PQB_DECODE_LUT = 1, 2, 4, 8
PQB_DECODE_PROBE_MEM, PQB_DECODE_PROBE_COMPUTE = 64, 128
PQB_DECODE_MERGE_KERNEL = 256
PQB_DECODE_NO_CLUSTER = 2048  # DQ kernel: no cluster / DSMEM split-merge path (A/B)
PQB_DECODE_MERGE_INKERNEL = 1024  # DQ kernel: force the in-launch split merge (A/B)
PQB_DECODE_DQ_LINEAR = 512  # DQ kernel: linear shared-memory layout build (automatic fallback)

c_i32, c_i64, c_u64, c_f32, c_f64, c_sz = (
    ctypes.c_int32,
    ctypes.c_int64,
    ctypes.c_uint64,
    ctypes.c_float,
    ctypes.c_double,
    ctypes.c_size_t,
)
c_vp = ctypes.c_void_p


class PqbStore(ctypes.Structure):
    _fields_ = [
        ("pool", c_vp),
        ("page_bytes", c_i64),
        ("angle_off", c_i64),
        ("radius_off", c_i64),
        ("value_off", c_i64),
        ("page_table", c_vp),
        ("max_pages", c_i32),
        ("page_tokens", c_i32),
        ("value_dtype", c_i32),
        ("reserved", c_i32),
    ]


class PqbCache(ctypes.Structure):
    _fields_ = [
        ("store", PqbStore),
        ("d", c_i32),
        ("angle_bits", c_i32),
        ("radius_bits", c_i32),
        ("layout", c_i32),
        ("scales", c_vp),
        ("seq_lens", c_vp),
        ("quant_lens", c_vp),
        ("residual", c_vp),
        ("res_cap", c_i32),
        ("reserved", c_i32),
    ]


PQB_MAX_PEERS = 8
PQB_IPC_HANDLE_BYTES = 64


class PqbPeerOut(ctypes.Structure):
    """pqb_peer_out (include/pqb200.h): the fused head-output gather of a layer."""

    _fields_ = [
        ("out", c_vp * PQB_MAX_PEERS),
        ("flags", c_vp * PQB_MAX_PEERS),
        ("n_peers", c_i32),
        ("rank", c_i32),
        ("batch0", c_i32),
        ("head0", c_i32),
        ("kv_local", c_i32),
        ("q_heads", c_i32),
        ("out_dtype", c_i32),
        ("reserved", c_i32),
    ]


# name -> (restype, argtypes); must match include/pqb200.h exactly
SIGNATURES: dict[str, tuple[object, list[object]]] = {
    "pqb_abi_version": (c_i32, []),
    "pqb_last_error": (ctypes.c_char_p, []),
    "pqb_device_count": (c_i32, []),
    "pqb_radius_scales": (
        c_i32,
        [c_vp, c_i32, c_i64, c_i64, c_i32, c_i64, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp],
    ),
    "pqb_encode": (
        c_i32,
        [c_vp, c_i32, c_i64, c_i64, c_i32, c_i64, c_i64, c_i32, c_i32, c_i32, c_vp,
         ctypes.POINTER(PqbStore), c_vp, c_i64, c_vp, c_vp, c_vp],
    ),
    "pqb_store_values": (
        c_i32,
        [c_vp, c_i32, c_i64, c_i64, c_i32, c_i64, c_i64, ctypes.POINTER(PqbStore), c_vp, c_i64, c_vp],
    ),
    "pqb_store_values_ex": (
        c_i32,
        [c_vp, c_i32, c_i64, c_i64, c_i32, c_i64, c_i64, ctypes.POINTER(PqbStore), c_vp, c_i64, c_vp, c_vp],
    ),
    "pqb_store_residual": (
        c_i32,
        [ctypes.POINTER(PqbCache), c_vp, c_i32, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp],
    ),
    "pqb_append": (
        c_i32,
        [ctypes.POINTER(PqbCache), c_i64, c_vp, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp],
    ),
    "pqb_decode_workspace_bytes": (c_sz, [c_i64, c_i32, c_i32, c_i32]),
    "pqb_decode_attn": (
        c_i32,
        [ctypes.POINTER(PqbCache), c_i64, c_i32, c_vp, c_i32, c_f32, c_i32, c_vp, c_i32, c_vp, c_i64,
         c_vp, c_sz, c_vp],
    ),
    "pqb_decode_attn_ex": (
        c_i32,
        [ctypes.POINTER(PqbCache), c_i64, c_i32, c_vp, c_i32, c_f32, c_i32, c_vp, c_i32, c_vp, c_i64,
         c_vp, c_sz, c_i32, c_i32, c_vp],
    ),
    "pqb_decode_splits": (c_i32, [c_i64, c_i32]),
    "pqb_decode_launches": (c_i32, [c_i64, c_i32, c_i32, c_i32]),
    "pqb_decode_launches_ex": (c_i32, [c_i64, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32]),
    "pqb_decode_dq_layout": (c_i32, []),
    "pqb_decode_split_starts": (c_i32, [c_i64, c_i32, c_i32, c_vp]),
    "pqb_decode_attn_peer": (
        c_i32,
        [ctypes.POINTER(PqbCache), c_i64, c_i32, c_vp, c_i32, c_f32, c_i32, ctypes.POINTER(PqbPeerOut), c_vp, c_sz,
         c_vp],
    ),
    "pqb_peer_wait": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_vp]),
    "pqb_ipc_alloc": (c_i32, [c_i32, c_sz, ctypes.POINTER(c_vp), c_vp]),
    "pqb_ipc_open": (c_i32, [c_i32, c_vp, ctypes.POINTER(c_vp)]),
    "pqb_ipc_close": (c_i32, [c_i32, c_vp]),
    "pqb_ipc_free": (c_i32, [c_i32, c_vp]),
    "pqb_peer_access": (c_i32, [c_i32, c_i32, ctypes.POINTER(c_i32)]),
    "pqb_angle_table": (c_i32, [c_i32, c_vp, c_vp, c_vp]),
    "pqb_query_lut": (c_i32, [c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "pqb_radius_table": (c_i32, [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp]),
    "pqb_unpack_codes": (
        c_i32,
        [ctypes.POINTER(PqbStore), c_i64, c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp],
    ),
    "pqb_export_streams": (
        c_i32,
        [ctypes.POINTER(PqbStore), c_i64, c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp],
    ),
    "pqb_pack_codes": (
        c_i32,
        [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, ctypes.POINTER(PqbStore), c_i64, c_vp],
    ),
    "pqb_read_values": (c_i32, [ctypes.POINTER(PqbStore), c_i64, c_i32, c_i64, c_vp, c_vp]),
    "pqb_dequantize": (
        c_i32,
        [ctypes.POINTER(PqbCache), c_i64, c_i64, c_vp, c_vp],
    ),
    "pqb_quantize_values": (c_i32, [c_vp, c_i32, c_i64, c_i32, c_i32, c_vp, c_vp]),
    "pqb_softmax_f64": (c_i32, [c_vp, c_i64, c_f64, c_vp, c_vp]),
    "pqb_to_polar": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_vp, c_vp, c_vp]),
    "pqb_quantize_angle": (c_i32, [c_vp, c_i32, c_i64, c_i32, c_vp, c_vp]),
    "pqb_angle_grid": (c_i32, [c_i32, c_vp, c_vp]),
    "pqb_quantize_radius": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "pqb_scores_direct": (c_i32, [ctypes.POINTER(PqbCache), c_i64, c_vp, c_i32, c_i64, c_vp, c_vp]),
    "pqb_import_streams": (
        c_i32,
        [ctypes.POINTER(PqbStore), c_i64, c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp],
    ),
    "pqb_synthetic_keys": (
        c_i32,
        [c_u64, c_i64, c_i64, c_i32, c_i32, c_f32, c_f32, c_u64, c_f32, c_vp, c_i32, c_vp],
    ),
    "pqb_synthetic_normal": (c_i32, [c_u64, c_i64, c_vp, c_i32, c_vp]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the library.  Raises RuntimeError if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # PQB_LIB: load another build of the same ABI (A/B timing of kernel variants)
        p = Path(path) if path else Path(os.environ.get("PQB_LIB", LIB_PATH))
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build the CUDA extension with "
                "`python -m paper_2502_00527_b200.build` (no CPU fallback exists)"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.pqb_abi_version() != 1:
            raise RuntimeError(f"libpqb200 ABI {lib.pqb_abi_version()} != 1")
        _lib = lib
        return lib


class PqbError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> None:
    """Map a PQB status to the exception the reference raises for that case."""
    if rc == PQB_OK:
        return
    msg = (load().pqb_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc in (PQB_EINVAL, PQB_EUNSUPPORTED):
        raise ValueError(text)
    raise RuntimeError(text)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
