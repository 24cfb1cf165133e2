"""The C-ABI boundary without a GPU: the library loads, exports exactly what
include/pqb200.h declares, the ctypes binding matches the header's arity, and
argument validation maps to the reference's exception types before any CUDA
work is enqueued."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from paper_2502_00527_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pqb200.h"


def declared() -> dict[str, int]:
    """name -> parameter count for every function prototype in the header."""
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    out = {}
    for m in re.finditer(r"\b(?:int|size_t|const char\*)\s+(pqb_\w+)\s*\(([^)]*)\)\s*;", text):
        params = m.group(2).strip()
        out[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_library_loads_and_reports_abi():
    lib = _lib.load()
    assert lib.pqb_abi_version() == 1
    assert lib.pqb_device_count() >= 0


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    names = declared()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name


def test_binding_matches_header_arity():
    names = declared()
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)
    for name, count in names.items():
        assert len(_lib.SIGNATURES[name][1]) == count, name


def test_struct_layout_matches_header():
    # pqb_store: 8 + 4*8 + 8 + 4*4 = 64 bytes; pqb_cache: store + 4*4 + 4*8 + 2*4
    assert ctypes.sizeof(_lib.PqbStore) == 64
    assert ctypes.sizeof(_lib.PqbCache) == 64 + 16 + 32 + 8
    # pqb_peer_out: 8 + 8 pointers, 8 int32
    assert ctypes.sizeof(_lib.PqbPeerOut) == 16 * 8 + 8 * 4


def test_peer_descriptor_validation():
    """A peer descriptor with a rank outside [0, n_peers) or a missing buffer is
    rejected before any CUDA work (ValueError)."""
    d = _lib.PqbPeerOut()
    d.n_peers, d.rank, d.kv_local, d.q_heads, d.out_dtype = 2, 2, 1, 8, 1
    rc = _lib.load().pqb_decode_attn_peer(None, 1, 8, None, 1, 1.0, 16, ctypes.byref(d), None, 0, None)
    assert rc == _lib.PQB_EINVAL
    d.rank = 0  # now the null buffers are the problem
    rc = _lib.load().pqb_decode_attn_peer(None, 1, 8, None, 1, 1.0, 16, ctypes.byref(d), None, 0, None)
    assert rc == _lib.PQB_EINVAL


@pytest.mark.parametrize(
    "call",
    [
        lambda L: L.pqb_radius_scales(None, 0, 1, 10, 7, 0, 0, 1, 4, None, None, None, None),  # odd d
        lambda L: L.pqb_radius_scales(None, 0, 1, 0, 8, 0, 0, 1, 4, None, None, None, None),  # empty
        lambda L: L.pqb_radius_scales(None, 0, 1, 10, 8, 0, 0, 1, 9, None, None, None, None),  # bits
        lambda L: L.pqb_encode(None, 0, 1, 1, 8, 0, 0, 1, 0, 4, None, None, None, 0, None, None, None),
        lambda L: L.pqb_query_lut(None, 0, 1, 8, 1, 4, None, None),
        lambda L: L.pqb_softmax_f64(None, 0, 1.0, None, None),  # empty score vector
        lambda L: L.pqb_angle_table(0, None, None, None),
        lambda L: L.pqb_peer_wait(None, 2, 0, None, None),  # null flags
        lambda L: L.pqb_decode_attn_peer(None, 1, 4, None, 1, 1.0, 16, None, None, 0, None),  # null peer
        lambda L: L.pqb_store_values_ex(None, 1, 1, 1, 7, 0, 0, None, None, 0, None, None),  # odd d
        lambda L: L.pqb_ipc_alloc(0, 0, None, None),  # null outputs, zero size
        lambda L: L.pqb_ipc_open(0, None, None),  # null handle
        lambda L: L.pqb_ipc_close(0, None),
        lambda L: L.pqb_ipc_free(0, None),
        lambda L: L.pqb_peer_access(0, 0, None),  # null output
    ],
)
def test_validation_maps_to_value_error(call):
    rc = call(_lib.load())
    assert rc in (_lib.PQB_EINVAL, _lib.PQB_EUNSUPPORTED)
    with pytest.raises(ValueError):
        _lib.check(rc, "x")
    assert _lib.load().pqb_last_error()


def test_state_errors_map_to_runtime_error():
    cache = _lib.PqbCache()  # no scales / lengths: "prefill first"
    rc = _lib.load().pqb_append(ctypes.byref(cache), 1, None, 0, None, 0, None, None, None)
    assert rc == _lib.PQB_ESTATE
    with pytest.raises(RuntimeError):
        _lib.check(rc)


def test_store_descriptor_validation():
    st = _lib.PqbStore(pool=1 << 20, page_bytes=4096, angle_off=0, radius_off=2048, value_off=-1,
                       page_table=None, max_pages=1, page_tokens=48, value_dtype=1, reserved=0)
    rc = _lib.load().pqb_unpack_codes(ctypes.byref(st), 0, 128, 4, 4, 1, None, None, None)
    assert rc == _lib.PQB_EINVAL  # page_tokens not a multiple of 32
    assert b"page_tokens" in _lib.load().pqb_last_error()


def test_balanced_split_host_logic():
    """The DQ kernel's cost-balanced persistent split (decode.cu
    make_split_balanced), host side only: CTA ranges cover the unit-major tile
    space exactly, in order, on no more CTAs than allowed; a range that crosses
    into a second unit is shorter than the single-unit ones (it pays a second
    setup and merge); short launches keep the uniform split."""
    lib = _lib.load()
    tm = 32768 // 32
    for units, ctas in [(128, 148), (32, 148), (64, 148), (128, 100), (5, 7)]:
        buf = (ctypes.c_int32 * (ctas + 1))()
        n = lib.pqb_decode_split_starts(units, 32768, ctas, buf)
        starts = list(buf)[: n + 1]
        assert 0 < n <= ctas
        assert starts[0] == 0 and starts[-1] == units * tm
        assert all(b > a for a, b in zip(starts, starts[1:]))
        one, two = [], []
        for a, b in zip(starts, starts[1:]):
            (two if (b - 1) // tm != a // tm else one).append(b - a)
        if one and two:
            assert max(two) < max(one)
    buf = (ctypes.c_int32 * 149)()
    assert lib.pqb_decode_split_starts(8, 4096, 148, buf) == 0  # configs[0]: a few tiles per CTA, uniform
    assert lib.pqb_decode_split_starts(8, 4096, 0, buf) == -1
