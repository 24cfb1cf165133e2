"""Paged polar key cache on the GPU.

``PolarKVCache``   batched store for n_units independent (layer, sequence,
                   kv-head) units: the layout the decode kernels stream.
``PackedKVCache``  the reference's single-head streaming cache API
                   (kv_cache.py:85-289) on top of a one-unit PolarKVCache.

HBM layout (one page = ``page_tokens`` tokens of one unit, 128-byte aligned):

    [ angle codes  P*(d/2)*m/8 B | radius codes P*(d/2)*n/8 B | values P*d*vb B ]

Angle/radius regions are byte slices of the reference code streams
(polar_codec.py:98-110), so concatenating a unit's pages reproduces
PolarCodes.angle_stream / radius_stream.  The page table maps (unit, page) to a
page id; scales are fp16 [U, d/2]; the residual window is an fp32 ring
[U, s, d] indexed by token % s (the reference's FIFO deque, kv_cache.py:107).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from ._device import (
    DTYPE_CODE,
    as_device_matrix,
    dtype_code,
    layout_code,
    new_flags,
    ptr,
    raise_on_flags,
    require_cuda,
    round_up,
    stream_ptr,
)
from .codec import encode_device, radius_scales_device
from .core import (
    BitReport,
    CacheSnapshot,
    ChannelScales,
    KeyTensor,
    PolarCodes,
    QuantConfig,
    stream_bytes,
)

SCALE_BITS = 16  # kv_cache.py:39
VQ_DTYPE = {2: _lib.PQB_VQ2, 4: _lib.PQB_VQ4, 8: _lib.PQB_VQ8}  # value_bits -> paged code layout
RESIDUAL_BITS = 16  # kv_cache.py:40


class PolarKVCache:
    """Batched paged polar-code + value cache for ``n_units`` units."""

    def __init__(
        self,
        cfg: QuantConfig,
        n_units: int,
        dim: int = 128,
        residual_len: int = 0,
        *,
        capacity: int = 1024,
        page_tokens: int = 128,
        value_dtype: torch.dtype = torch.bfloat16,
        device=None,
        shuffle_pages: bool = False,
        seed: int = 0,
        value_bits: int | None = None,
    ) -> None:
        if residual_len < 0:
            raise ValueError(f"residual_len must be >= 0, got {residual_len}")
        if dim < 2 or dim % 2:
            raise ValueError(f"dim must be even and >= 2, got {dim}")
        if page_tokens <= 0 or page_tokens % 32:
            raise ValueError(f"page_tokens must be a positive multiple of 32, got {page_tokens}")
        if value_dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("value_dtype must be torch.float32 or torch.bfloat16")
        if value_bits is not None:
            # per-token uniform value codes (PackedKVCache(quantize_values=True), kv_cache.py:199-209)
            if not 1 <= int(value_bits) <= 8:
                raise ValueError(f"bits must be in [1, 8], got {value_bits}")
            if int(value_bits) not in VQ_DTYPE or dim != 128:
                raise ValueError("the batched cache stores quantized values as 2-, 4- or 8-bit codes with dim = 128 "
                                 f"(got value_bits={value_bits}, dim={dim}); PackedKVCache keeps other widths "
                                 "as their dequantized fp32 rows")
        self.device = require_cuda(device)
        self.cfg = cfg
        self.n_units = int(n_units)
        self.dim = int(dim)
        self.residual_len = int(residual_len)
        self.page_tokens = int(page_tokens)
        self.value_dtype = value_dtype
        self.value_bits = None if value_bits is None else int(value_bits)
        self.shuffle_pages = shuffle_pages
        self._seed = seed
        half = dim // 2
        P = self.page_tokens
        a_bytes = P * half * cfg.angle_bits // 8
        r_bytes = P * half * cfg.radius_bits // 8
        if self.value_bits is not None:
            v_bytes = P * 16 * self.value_bits + P * 8  # b-bit codes (MMA-fragment order) + (zp, scale) fp32 per token
        else:
            v_bytes = P * dim * (4 if value_dtype == torch.float32 else 2)
        self.angle_off = 0
        self.radius_off = round_up(a_bytes, 128)
        self.value_off = round_up(self.radius_off + r_bytes, 128)
        self.page_bytes = round_up(self.value_off + v_bytes, 128)
        dev = self.device
        U = self.n_units
        self.scales16 = torch.zeros((U, half), dtype=torch.float16, device=dev)
        self.seq_lens = torch.zeros(U, dtype=torch.int32, device=dev)
        self.quant_lens = torch.zeros(U, dtype=torch.int32, device=dev)
        self.clamp_counts = torch.zeros(U, dtype=torch.int64, device=dev)
        self.flags = new_flags(dev)
        self.residual = (
            torch.zeros((U, residual_len, dim), dtype=torch.float32, device=dev) if residual_len else None
        )
        self._scale_ws = torch.empty(U * half, dtype=torch.int64, device=dev)
        self.host_seq = np.zeros(U, dtype=np.int64)
        self.host_quant = np.zeros(U, dtype=np.int64)
        self._filled = np.zeros(U, dtype=bool)
        self._all_view: UnitView | None = None
        self.prefilled = False
        self.max_pages = 0
        self._gen = 0  # storage generation: bumped whenever pool / page_table are replaced
        self._alloc(max(int(capacity), 1))

    # ------------------------------------------------------------ storage

    def _alloc(self, capacity: int) -> None:
        max_pages = math.ceil(capacity / self.page_tokens)
        U = self.n_units
        pool = torch.zeros(U * max_pages * self.page_bytes, dtype=torch.uint8, device=self.device)
        if self.shuffle_pages:
            g = torch.Generator().manual_seed(self._seed)
            perm = torch.randperm(U * max_pages, generator=g).to(torch.int32)
            table = perm.view(U, max_pages).to(self.device)
        else:
            table = torch.arange(U * max_pages, dtype=torch.int32, device=self.device).view(U, max_pages)
        if self.max_pages:  # grow: copy old pages (identity tables only)
            old = self.pool.view(U, self.max_pages, self.page_bytes)
            pool.view(U, max_pages, self.page_bytes)[:, : self.max_pages].copy_(old)
        self.pool, self.page_table, self.max_pages = pool, table.contiguous(), max_pages
        self._gen += 1  # views built before this re-derive their descriptors (UnitView._sync)
        self._rebuild_struct()

    def _rebuild_struct(self) -> None:
        store = _lib.PqbStore(
            pool=ptr(self.pool),
            page_bytes=self.page_bytes,
            angle_off=self.angle_off,
            radius_off=self.radius_off,
            value_off=self.value_off,
            page_table=ptr(self.page_table),
            max_pages=self.max_pages,
            page_tokens=self.page_tokens,
            value_dtype=(VQ_DTYPE[self.value_bits] if self.value_bits is not None
                         else _lib.PQB_F32 if self.value_dtype == torch.float32 else _lib.PQB_BF16),
            reserved=0,
        )
        self._struct = _lib.PqbCache(
            store=store,
            d=self.dim,
            angle_bits=self.cfg.angle_bits,
            radius_bits=self.cfg.radius_bits,
            layout=layout_code(self.cfg.layout),
            scales=ptr(self.scales16),
            seq_lens=ptr(self.seq_lens),
            quant_lens=ptr(self.quant_lens),
            residual=ptr(self.residual),
            res_cap=self.residual_len,
            reserved=0,
        )

    @property
    def capacity(self) -> int:
        return self.max_pages * self.page_tokens

    def ensure_capacity(self, tokens: int) -> None:
        if tokens > self.capacity:
            if self.shuffle_pages:
                raise RuntimeError("capacity exceeded on a cache with a shuffled page table")
            self._alloc(max(tokens, int(self.capacity * 1.5)))

    def cache_ref(self):
        return ctypes.byref(self._struct)

    def store_ref(self):
        return ctypes.byref(self._struct.store)

    def sub_struct(self, u0: int, u1: int) -> _lib.PqbCache:
        """Descriptor of units [u0, u1): every per-unit pointer offset by u0."""
        if not 0 <= u0 < u1 <= self.n_units:
            raise ValueError(f"bad unit range [{u0}, {u1})")
        s = _lib.PqbCache.from_buffer_copy(self._struct)
        s.store.page_table = ptr(self.page_table[u0])
        s.scales = ptr(self.scales16[u0])
        s.seq_lens = ptr(self.seq_lens[u0:])
        s.quant_lens = ptr(self.quant_lens[u0:])
        if self.residual is not None:
            s.residual = ptr(self.residual[u0])
        return s

    def view(self, u0: int, u1: int) -> "UnitView":
        """Decode-only view of units [u0, u1) (e.g. one layer of a multi-layer cache)."""
        return UnitView(self, u0, u1)

    @property
    def bytes_per_token(self) -> int:
        half = self.dim // 2
        if self.value_bits is not None:
            return half * (self.cfg.angle_bits + self.cfg.radius_bits) // 8 + 16 * self.value_bits + 8
        vb = 4 if self.value_dtype == torch.float32 else 2
        return half * (self.cfg.angle_bits + self.cfg.radius_bits) // 8 + self.dim * vb

    # -------------------------------------------------------------- writes

    def _prepare(self, x, what: str) -> torch.Tensor:
        t = as_device_matrix(x, self.device)
        if t.dtype not in DTYPE_CODE:
            raise ValueError(f"{what}: unsupported dtype {t.dtype}")
        return t

    def prefill(self, keys, values=None, *, unit_start: int = 0, check: bool = True) -> None:
        """Scale fit + bulk encode of [k, T, d] prompts into units
        [unit_start, unit_start + k) (kv_cache.py:152-177).

        The newest residual_len tokens of every unit stay in the fp32 ring.
        The cache counts as prefilled once every unit has been filled."""
        k = self._prepare(keys, "keys")
        if k.dim() == 2 and self.n_units == 1:
            k = k.unsqueeze(0)
        if k.dim() != 3 or k.shape[2] != self.dim:
            raise ValueError(f"keys must be [units, T, {self.dim}], got {tuple(k.shape)}")
        u0, u1 = unit_start, unit_start + k.shape[0]
        if not 0 <= u0 < u1 <= self.n_units:
            raise ValueError(f"units [{u0}, {u1}) outside [0, {self.n_units})")
        if self.prefilled or self._filled[u0:u1].any():
            raise RuntimeError("cache already prefilled")
        T = k.shape[1]
        if T == 0:
            raise ValueError("cannot compute scales from an empty tensor")
        v = None
        if values is not None:
            v = self._prepare(values, "values")
            if v.dim() == 2 and self.n_units == 1:
                v = v.unsqueeze(0)
            if tuple(v.shape) != tuple(k.shape):
                raise ValueError(f"values shape {tuple(v.shape)} != {tuple(k.shape)}")
        self.ensure_capacity(T)
        sub = self.sub_struct(u0, u1)
        sref = ctypes.byref(sub)
        n = u1 - u0
        flags = new_flags(self.device)  # this call's faults only (self.flags keeps the unchecked ones)
        radius_scales_device(k, self.cfg, flags, self._scale_ws, out=self.scales16[u0:u1])
        boundary = max(0, T - self.residual_len)
        if boundary:
            encode_device(k[:, :boundary], self.scales16[u0:u1], self.cfg, ctypes.byref(sub.store),
                          clamp_counts=self.clamp_counts[u0:u1], flags=flags)
        if T > boundary:
            kr = k[:, boundary:]
            if kr.stride(-1) != 1:
                kr = kr.contiguous()
            _lib.call("pqb_store_residual", sref, ptr(kr), dtype_code(kr), n, T - boundary,
                      kr.stride(0), kr.stride(1), boundary, ptr(flags), stream_ptr(self.device))
        if v is not None and v.stride(-1) != 1:
            v = v.contiguous()
        _lib.call(
            "pqb_store_values_ex", ptr(v), dtype_code(v) if v is not None else 0, n, T, self.dim,
            v.stride(0) if v is not None else 0, v.stride(1) if v is not None else 0, ctypes.byref(sub.store),
            None, 0, ptr(flags), stream_ptr(self.device),
        )
        self.seq_lens[u0:u1].fill_(T)
        self.quant_lens[u0:u1].fill_(boundary)
        self.host_seq[u0:u1] = T
        self.host_quant[u0:u1] = boundary
        self._filled[u0:u1] = True
        self.prefilled = bool(self._filled.all())
        if check:
            try:
                raise_on_flags(flags, "prefill")
            except ValueError:
                self._reset_units(u0, u1)  # units filled by earlier calls are kept
                raise
        else:
            self.flags.bitwise_or_(flags)  # reported by check()

    def import_unit(self, unit: int, codes: PolarCodes, scales: ChannelScales, residual_keys=None,
                    clamp_events: int = 0, values=None) -> None:
        """Load one unit from reference containers (load_codes / load_snapshot,
        polar_codec.py:415-446, kv_cache.py:369-397): the two code streams are
        scattered into the unit's pages (pqb_import_streams), the residual keys
        (oldest first) fill the ring after them, values default to zeros.  The
        unit then decodes and streams like a prefilled one."""
        if not 0 <= unit < self.n_units:
            raise ValueError(f"unit {unit} outside [0, {self.n_units})")
        if self._filled[unit]:
            raise RuntimeError("cache already prefilled")
        cfg = codes.config()
        if (cfg.angle_bits, cfg.radius_bits, cfg.layout) != (self.cfg.angle_bits, self.cfg.radius_bits,
                                                             self.cfg.layout):
            raise ValueError(f"codes config {cfg} does not match cache config {self.cfg}")
        if codes.dim != self.dim or scales.num_channels != self.dim // 2:
            raise ValueError(f"codes dim {codes.dim} / {scales.num_channels} scales != cache dim {self.dim}")
        res = np.zeros((0, self.dim), np.float32) if residual_keys is None else np.asarray(residual_keys, np.float32)
        if res.ndim != 2 or res.shape[1] != self.dim:
            raise ValueError(f"residual keys must be (k, {self.dim}), got {res.shape}")
        if res.shape[0] > self.residual_len:
            raise ValueError(f"{res.shape[0]} residual keys exceed the window of {self.residual_len}")
        Tq = codes.num_tokens
        T = Tq + res.shape[0]
        self.ensure_capacity(T)
        sub = self.sub_struct(unit, unit + 1)
        dev = self.device
        if Tq:
            a = torch.frombuffer(bytearray(codes.angle_stream), dtype=torch.uint8).to(dev)
            r = torch.frombuffer(bytearray(codes.radius_stream), dtype=torch.uint8).to(dev)
            _lib.call("pqb_import_streams", self.store_ref(), unit, self.dim, cfg.angle_bits, cfg.radius_bits, Tq,
                      ptr(a), ptr(r), stream_ptr(dev))
        self.scales16[unit] = torch.from_numpy(np.array(scales.values, dtype=np.float16)).to(dev)
        flags = new_flags(dev)
        if res.shape[0]:
            kr = torch.from_numpy(res).to(dev).unsqueeze(0)
            _lib.call("pqb_store_residual", ctypes.byref(sub), ptr(kr), _lib.PQB_F32, 1, res.shape[0],
                      kr.stride(0), kr.stride(1), Tq, ptr(flags), stream_ptr(dev))
        v = None
        if values is not None:
            v = as_device_matrix(values, dev).reshape(1, T, self.dim).contiguous()
        if T:
            _lib.call("pqb_store_values_ex", ptr(v), dtype_code(v) if v is not None else 0, 1, T, self.dim,
                      v.stride(0) if v is not None else 0, v.stride(1) if v is not None else 0,
                      ctypes.byref(sub.store), None, 0, ptr(flags), stream_ptr(dev))
        self.seq_lens[unit] = T
        self.quant_lens[unit] = Tq
        self.clamp_counts[unit] = int(clamp_events)
        self.host_seq[unit] = T
        self.host_quant[unit] = Tq
        self._filled[unit] = True
        self.prefilled = bool(self._filled.all())
        try:
            raise_on_flags(flags, "import")
        except ValueError:
            self._reset_units(unit, unit + 1)
            raise

    def snapshot_unit(self, unit: int = 0) -> CacheSnapshot:
        """CacheSnapshot of one unit (kv_cache.py:261-268): packed streams
        gathered from the pages, scales, residual keys oldest first."""
        return CacheSnapshot(codes=self.export_codes(unit), scales=ChannelScales(self.scales16[unit].cpu().numpy()),
                             residual_keys=self.residual_keys(unit).cpu().numpy(), residual_len=self.residual_len,
                             clamp_events=int(self.clamp_counts[unit].item()))

    def append(self, keys, values=None, *, check: bool = False) -> None:
        """One streaming token per unit (kv_cache.py:179-189): keys/values [U, d]."""
        if not self.prefilled:
            raise RuntimeError("cache is empty; prefill first")
        k = self._prepare(keys, "key")
        if k.dim() == 1 and self.n_units == 1:
            k = k.unsqueeze(0)
        if k.dim() != 2 or k.shape[0] != self.n_units or k.shape[1] != self.dim:
            raise ValueError(f"key dim {tuple(k.shape)} != cache dim ({self.n_units}, {self.dim})")
        k = k.contiguous()
        v = None
        if values is not None:
            v = self._prepare(values, "value").reshape(self.n_units, self.dim).contiguous()
        self.ensure_capacity(int(self.host_seq.max()) + 2)
        flags = new_flags(self.device) if check else self.flags  # unchecked faults stay for check()
        _lib.call("pqb_append", self.cache_ref(), self.n_units, ptr(k), dtype_code(k), ptr(v),
                  dtype_code(v) if v is not None else 0, ptr(self.clamp_counts), ptr(flags),
                  stream_ptr(self.device))
        flush = (self.host_seq - self.host_quant) >= self.residual_len
        self.host_quant = self.host_quant + flush.astype(np.int64)
        self.host_seq = self.host_seq + 1
        if check:  # the token is committed either way (the reference's append does not validate)
            raise_on_flags(flags, "append")

    def check(self) -> None:
        """Raise ValueError if any unchecked prefill / append so far saw a
        non-finite key or an fp16 scale overflow (synchronizes); clears the word."""
        try:
            raise_on_flags(self.flags, "cache")
        finally:
            self.flags.zero_()

    def _reset_units(self, u0: int, u1: int) -> None:
        """Return units [u0, u1) to the empty state: zero their pages (the
        encoder ORs codes into fresh pages), lengths, scales and residual rows."""
        ids = self.page_table[u0:u1].reshape(-1).long()
        self.pool.view(-1, self.page_bytes).index_fill_(0, ids, 0)
        self.seq_lens[u0:u1] = 0
        self.quant_lens[u0:u1] = 0
        self.clamp_counts[u0:u1] = 0
        self.scales16[u0:u1] = 0
        if self.residual is not None:
            self.residual[u0:u1] = 0
        self.host_seq[u0:u1] = 0
        self.host_quant[u0:u1] = 0
        self._filled[u0:u1] = False
        self.prefilled = False

    def reset(self) -> None:
        self.pool.zero_()
        self.seq_lens.zero_()
        self.quant_lens.zero_()
        self.clamp_counts.zero_()
        self.flags.zero_()
        if self.residual is not None:
            self.residual.zero_()
        self.host_seq[:] = 0
        self.host_quant[:] = 0
        self._filled[:] = False
        self.prefilled = False

    # ------------------------------------------------------------ decode

    def _all(self) -> "UnitView":
        if self._all_view is None:
            self._all_view = UnitView(self, 0, self.n_units)
        return self._all_view

    def decode(self, q, sm_scale: float | None = None, **kw) -> torch.Tensor:
        """softmax(q K^T * sm_scale) V for every unit, q [U, G, d] -> [U, G, d].

        K^T is the LUT score of qk_scores (bit-identical in fp32); sm_scale
        defaults to 1/sqrt(d) (cli.py:297's temperature)."""
        return self._all().decode(q, sm_scale, **kw)

    def scores(self, q, max_tokens: int | None = None) -> torch.Tensor:
        """LUT scores [U, G, T_max] fp32 (qk_scores, lut_decode.py:119-154);
        entries beyond a unit's length are left unset."""
        return self._all().scores(q, max_tokens)

    # ----------------------------------------------------------- readers

    def code_arrays(self, unit: int = 0) -> tuple[torch.Tensor, torch.Tensor]:
        Tq = int(self.host_quant[unit])
        half = self.dim // 2
        a = torch.empty((Tq, half), dtype=torch.uint8, device=self.device)
        r = torch.empty((Tq, half), dtype=torch.uint8, device=self.device)
        if Tq:
            _lib.call("pqb_unpack_codes", self.store_ref(), unit, self.dim, self.cfg.angle_bits,
                      self.cfg.radius_bits, Tq, ptr(a), ptr(r), stream_ptr(self.device))
        return a, r

    def export_codes(self, unit: int = 0) -> PolarCodes:
        Tq = int(self.host_quant[unit])
        count = Tq * (self.dim // 2)
        na, nr = stream_bytes(count, self.cfg.angle_bits), stream_bytes(count, self.cfg.radius_bits)
        a = torch.empty(max(na, 1), dtype=torch.uint8, device=self.device)
        r = torch.empty(max(nr, 1), dtype=torch.uint8, device=self.device)
        if Tq:
            _lib.call("pqb_export_streams", self.store_ref(), unit, self.dim, self.cfg.angle_bits,
                      self.cfg.radius_bits, Tq, ptr(a), ptr(r), stream_ptr(self.device))
        return PolarCodes(Tq, self.dim, self.cfg.angle_bits, self.cfg.radius_bits, self.cfg.layout,
                          a[:na].cpu().numpy().tobytes(), r[:nr].cpu().numpy().tobytes())

    def values_f32(self, unit: int = 0) -> torch.Tensor:
        T = int(self.host_seq[unit])
        out = torch.empty((T, self.dim), dtype=torch.float32, device=self.device)
        if T:
            _lib.call("pqb_read_values", self.store_ref(), unit, self.dim, T, ptr(out), stream_ptr(self.device))
        return out

    def residual_keys(self, unit: int = 0) -> torch.Tensor:
        T, Tq = int(self.host_seq[unit]), int(self.host_quant[unit])
        if T == Tq or self.residual is None:
            return torch.zeros((0, self.dim), dtype=torch.float32, device=self.device)
        slots = torch.arange(Tq, T, device=self.device) % self.residual_len
        return self.residual[unit, slots]

    def dequantize(self, unit: int = 0) -> torch.Tensor:
        """Quantized region of one unit as fp32 keys (decode_quantized, kv_cache.py:239-245)."""
        Tq = int(self.host_quant[unit])
        out = torch.empty((Tq, self.dim), dtype=torch.float32, device=self.device)
        if Tq:
            _lib.call("pqb_dequantize", self.cache_ref(), unit, Tq, ptr(out), stream_ptr(self.device))
        return out

    def scores_direct(self, q: torch.Tensor, unit: int = 0, tokens: int | None = None) -> torch.Tensor:
        """qk_scores_direct of one unit (lut_decode.py:157-186): dequantized keys
        dotted with q [d] in fp32, then the residual keys; fp32 [T]."""
        T = int(self.host_seq[unit]) if tokens is None else int(tokens)
        out = torch.empty(max(T, 0), dtype=torch.float32, device=self.device)
        if T:
            _lib.call("pqb_scores_direct", self.cache_ref(), unit, ptr(q), dtype_code(q), T, ptr(out),
                      stream_ptr(self.device))
        return out

    def radius_table(self) -> torch.Tensor:
        half = self.dim // 2
        L = self.cfg.radius_levels
        out = torch.empty((self.n_units, half, L), dtype=torch.float32, device=self.device)
        _lib.call("pqb_radius_table", ptr(self.scales16), self.n_units, self.dim, self.cfg.radius_bits, ptr(out),
                  stream_ptr(self.device))
        return out


class UnitView:
    """Decode entry for units [u0, u1) of a PolarKVCache (e.g. one layer).

    Holds its own C descriptor so repeated calls need no per-call host work
    beyond argument marshalling.  The descriptor is re-derived whenever the
    cache has replaced its pool / page table (growth on append), so a view
    never reads freed storage.  A CUDA graph captured before such a growth
    still holds the old pointers and must be re-captured."""

    def __init__(self, cache: PolarKVCache, u0: int, u1: int) -> None:
        self.cache = cache
        self.u0, self.u1 = u0, u1
        self.n_units = u1 - u0
        self._ws: torch.Tensor | None = None
        self._gen = -1
        self._sync()

    def _sync(self) -> None:
        if self._gen != self.cache._gen:
            self.struct = self.cache.sub_struct(self.u0, self.u1)
            self.ref = ctypes.byref(self.struct)
            self._gen = self.cache._gen

    def workspace(self, group: int, max_tokens: int) -> torch.Tensor:
        """Per-view decode workspace.  Zero-filled once: its leading counter
        region (split-merge bookkeeping) is left zeroed by every call."""
        need = _lib.load().pqb_decode_workspace_bytes(self.n_units, group, max_tokens, self.cache.dim)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(max(need, 256), dtype=torch.uint8, device=self.cache.device)
        return self._ws

    @property
    def max_tokens(self) -> int:
        return int(self.cache.host_seq[self.u0 : self.u1].max())

    def _t_max(self, max_tokens: int | None) -> int:
        """Tile bound of a launch: the view's longest unit, or a caller bound
        (e.g. a graph captured at capacity) that must not be below it -- the
        kernels cut each unit's tiles at this bound and size score rows by it."""
        actual = self.max_tokens
        if max_tokens is None:
            return actual
        if int(max_tokens) < actual:
            raise ValueError(f"max_tokens={int(max_tokens)} is below the longest unit's {actual} tokens")
        return int(max_tokens)

    def _check_q(self, q) -> torch.Tensor:
        c = self.cache
        self._sync()
        if not c._filled[self.u0 : self.u1].all():
            raise RuntimeError("cache is empty; prefill first")
        q = as_device_matrix(q, c.device)
        if q.dim() != 3 or q.shape[0] != self.n_units or q.shape[2] != c.dim:
            raise ValueError(f"query must be [{self.n_units}, G, {c.dim}], got {tuple(q.shape)}")
        return q if q.is_contiguous() else q.contiguous()

    def decode(self, q, sm_scale: float | None = None, *, out_dtype: torch.dtype = torch.float32,
               out: torch.Tensor | None = None, scores: torch.Tensor | None = None,
               max_tokens: int | None = None, flags: int = 0, splits: int = 0) -> torch.Tensor:
        c = self.cache
        q = self._check_q(q)
        G = q.shape[1]
        T_max = self._t_max(max_tokens)
        if T_max <= 0:
            raise ValueError("cannot attend over an empty cache")
        if out is None:
            out = torch.empty((self.n_units, G, c.dim), dtype=out_dtype, device=c.device)
        ws = self.workspace(G, T_max)
        scale = (1.0 / math.sqrt(c.dim)) if sm_scale is None else float(sm_scale)
        _lib.call(
            "pqb_decode_attn_ex", self.ref, self.n_units, G, ptr(q), dtype_code(q), scale, T_max, ptr(out),
            dtype_code(out), ptr(scores), scores.shape[-1] if scores is not None else 0, ptr(ws), ws.numel(),
            flags, splits, stream_ptr(c.device),
        )
        return out

    def decode_peer(self, q, peer: "_lib.PqbPeerOut", sm_scale: float | None = None,
                    max_tokens: int | None = None) -> None:
        """Fused decode + head-output gather (pqb_decode_attn_peer): outputs go
        straight into every peer's gathered buffer described by ``peer``."""
        c = self.cache
        q = self._check_q(q)
        G = q.shape[1]
        T_max = self._t_max(max_tokens)
        if T_max <= 0:
            raise ValueError("cannot attend over an empty cache")
        ws = self.workspace(G, T_max)
        scale = (1.0 / math.sqrt(c.dim)) if sm_scale is None else float(sm_scale)
        _lib.call("pqb_decode_attn_peer", self.ref, self.n_units, G, ptr(q), dtype_code(q), scale, T_max,
                  ctypes.byref(peer), ptr(ws), ws.numel(), stream_ptr(c.device))

    def scores(self, q, max_tokens: int | None = None, *, flags: int = 0,
               out: torch.Tensor | None = None) -> torch.Tensor:
        c = self.cache
        q = self._check_q(q)
        G = q.shape[1]
        T_max = self._t_max(max_tokens)
        if out is not None:
            if (out.dtype != torch.float32 or out.dim() != 3 or tuple(out.shape[:2]) != (self.n_units, G)
                    or out.shape[2] < T_max or out.stride(2) != 1 or out.stride(1) != out.shape[2]
                    or out.stride(0) != G * out.shape[2]):
                raise ValueError(f"out must be a contiguous float32 [{self.n_units}, {G}, >= {T_max}] tensor")
            sc = out
        else:
            sc = torch.empty((self.n_units, G, max(T_max, 1)), dtype=torch.float32, device=c.device)
        if T_max > 0:
            _lib.call(
                "pqb_decode_attn_ex", self.ref, self.n_units, G, ptr(q), dtype_code(q), 1.0, T_max, None, 0,
                ptr(sc), sc.shape[-1], None, 0, flags, 0, stream_ptr(c.device),
            )
        return sc[:, :, :T_max]


class PackedKVCache:
    """Token-streaming key cache storing polar codes plus a residual FIFO.

    Drop-in for polarquant.kv_cache.PackedKVCache (kv_cache.py:85-289): same
    constructor, methods, return types and exceptions; state lives on the GPU."""

    def __init__(self, cfg: QuantConfig, residual_len: int, *, quantize_values: bool = False,
                 value_bits: int = 4, device=None) -> None:
        if residual_len < 0:
            raise ValueError(f"residual_len must be >= 0, got {residual_len}")
        self.cfg = cfg
        self.residual_len = residual_len
        self.quantize_values = quantize_values
        self.value_bits = value_bits
        self._device = device
        self._dev: PolarKVCache | None = None
        self._dim: int | None = None
        self._consolidated = None
        self._radius_table = None

    # -- state -----------------------------------------------------------

    @property
    def prefilled(self) -> bool:
        return self._dev is not None and self._dev.prefilled

    @property
    def dim(self) -> int:
        if self._dim is None:
            raise RuntimeError("cache is empty; prefill first")
        return self._dim

    @property
    def scales(self) -> ChannelScales:
        if not self.prefilled:
            raise RuntimeError("cache is empty; prefill first")
        return ChannelScales(self._dev.scales16[0].cpu().numpy())

    @property
    def quantized_tokens(self) -> int:
        return int(self._dev.host_quant[0]) if self.prefilled else 0

    @property
    def residual_tokens(self) -> int:
        return int(self._dev.host_seq[0] - self._dev.host_quant[0]) if self.prefilled else 0

    @property
    def num_tokens(self) -> int:
        return self.quantized_tokens + self.residual_tokens

    @property
    def clamp_events(self) -> int:
        return int(self._dev.clamp_counts[0].item()) if self._dev is not None else 0

    @clamp_events.setter
    def clamp_events(self, value: int) -> None:
        if self._dev is None:
            raise RuntimeError("cache is empty; prefill first")
        self._dev.clamp_counts[0] = int(value)

    @property
    def residual_keys(self) -> np.ndarray:
        if not self.prefilled:
            d = self._dim if self._dim is not None else 0
            return np.zeros((0, d), dtype=np.float32)
        return self._dev.residual_keys(0).cpu().numpy()

    @property
    def device_cache(self) -> PolarKVCache:
        if self._dev is None:
            raise RuntimeError("cache is empty; prefill first")
        return self._dev

    @classmethod
    def from_snapshot(cls, snap: CacheSnapshot, device=None) -> "PackedKVCache":
        """A prefilled cache restored from a snapshot (load_snapshot,
        kv_cache.py:363-397): codes, scales, residual window and clamp count;
        values are zeros; further appends continue the stream."""
        cache = cls(snap.codes.config(), snap.residual_len, device=device)
        dev = require_cuda(device)
        d = snap.codes.dim
        T = snap.codes.num_tokens + np.asarray(snap.residual_keys).shape[0]
        cache._dim = d
        cache._dev = PolarKVCache(cache.cfg, 1, d, snap.residual_len, capacity=max(T + 64, 128), page_tokens=64,
                                  value_dtype=torch.float32, device=dev)
        try:
            cache._dev.import_unit(0, snap.codes, snap.scales, snap.residual_keys, snap.clamp_events)
        except Exception:
            cache._dev = None
            cache._dim = None
            raise
        return cache

    # -- writes ----------------------------------------------------------

    def _value_rows(self, values, count: int) -> torch.Tensor | None:
        if values is None:
            return None
        dev = self._dev.device
        v = as_device_matrix(np.asarray(values, dtype=np.float32) if not isinstance(values, torch.Tensor) else values,
                             dev)
        if tuple(v.shape) != (count, self._dim):
            raise ValueError(f"values shape {tuple(v.shape)} != ({count}, {self._dim})")
        if self.quantize_values:
            if not 1 <= self.value_bits <= 8:
                raise ValueError(f"bits must be in [1, 8], got {self.value_bits}")
            if not bool(torch.isfinite(v).all()):  # quantize_uniform, baseline_quant.py:88-89 (before any write)
                raise ValueError("values contain non-finite entries")
            if self._dev.value_bits is not None:  # code pages: the store kernel quantizes
                return v.to(torch.float32)
            out = torch.empty((count, self._dim), dtype=torch.float32, device=dev)
            v = v.contiguous()
            _lib.call("pqb_quantize_values", ptr(v), dtype_code(v), count, self._dim, self.value_bits, ptr(out),
                      stream_ptr(dev))
            return out
        return v.to(torch.float32)

    def prefill(self, keys: KeyTensor | np.ndarray, values: np.ndarray | None = None) -> None:
        if self.prefilled:
            raise RuntimeError("cache already prefilled")
        dev = require_cuda(self._device)
        m = as_device_matrix(keys, dev)
        if m.dim() != 2:
            raise ValueError(f"keys must be 2-D, got shape {tuple(m.shape)}")
        T, d = m.shape
        if d < 2 or d % 2:
            raise ValueError(f"vector dimension must be even and >= 2, got {d}")
        self._dim = d
        # quantized values of 2 / 4 / 8 bits at d = 128 live as code pages (the
        # decode kernel reads them); other widths as their dequantized fp32 rows
        vq = self.quantize_values and self.value_bits in VQ_DTYPE and d == 128
        self._dev = PolarKVCache(self.cfg, 1, d, self.residual_len, capacity=max(T + 64, 128), page_tokens=64,
                                 value_dtype=torch.float32, device=dev, value_bits=self.value_bits if vq else None)
        try:
            v = self._value_rows(values, T)
            if values is None and self.quantize_values:
                v = self._value_rows(np.zeros((T, d), dtype=np.float32), T)
            self._dev.prefill(m.unsqueeze(0), None if v is None else v.unsqueeze(0))
        except Exception:
            self._dev = None
            self._dim = None
            raise
        self._consolidated = None

    def append(self, key: np.ndarray, value: np.ndarray | None = None) -> None:
        if not self.prefilled:
            raise RuntimeError("cache is empty; prefill first")
        dev = self._dev.device
        row = as_device_matrix(np.asarray(key, dtype=np.float32).reshape(-1)
                               if not isinstance(key, torch.Tensor) else key.reshape(-1), dev)
        if row.shape[0] != self._dim:
            raise ValueError(f"key dim {row.shape[0]} != cache dim {self._dim}")
        v = None
        if value is not None:
            v = self._value_rows(np.asarray(value).reshape(1, -1) if not isinstance(value, torch.Tensor)
                                 else value.reshape(1, -1), 1)
        elif self.quantize_values:
            v = self._value_rows(np.zeros((1, self._dim), dtype=np.float32), 1)
        # the reference's append does not validate keys (kv_cache.py:179-189): a
        # non-finite key is committed like any other, and later appends still work
        self._dev.append(row.unsqueeze(0), v, check=False)
        self._consolidated = None

    # -- reads -----------------------------------------------------------

    def code_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        if self._consolidated is None:
            if not self.prefilled:
                half = (self._dim or 2) // 2
                empty = np.zeros((0, half), dtype=np.uint8)
                return empty, empty
            a, r = self._dev.code_arrays(0)
            self._consolidated = (a.cpu().numpy(), r.cpu().numpy())
        return self._consolidated

    @property
    def quantized(self) -> PolarCodes:
        return self.device_cache.export_codes(0)

    def radius_table(self) -> np.ndarray:
        if self._radius_table is None:
            self._radius_table = self.device_cache.radius_table()[0].cpu().numpy()
        return self._radius_table

    def decode_quantized(self) -> np.ndarray:
        return self.device_cache.dequantize(0).cpu().numpy()

    def values(self) -> np.ndarray:
        if not self.prefilled:
            d = self._dim if self._dim is not None else 0
            return np.zeros((0, d), dtype=np.float32)
        return self._dev.values_f32(0).cpu().numpy()

    def snapshot(self) -> CacheSnapshot:
        return CacheSnapshot(
            codes=self.quantized,
            scales=self.scales,
            residual_keys=self.residual_keys,
            residual_len=self.residual_len,
            clamp_events=self.clamp_events,
        )

    def memory_report(self) -> BitReport:
        """Bit accounting (kv_cache.py:270-289)."""
        if not self.prefilled:
            return BitReport(0, 0, 0, 0.0, 0.0, 0, 0, 0)
        tq, tr = self.quantized_tokens, self.residual_tokens
        total = tq + tr
        d = self.dim
        half = d // 2
        payload = tq * half * (self.cfg.angle_bits + self.cfg.radius_bits)
        params = half * SCALE_BITS
        residual = tr * d * RESIDUAL_BITS
        avg = (payload + params + residual) / (total * d) if total else 0.0
        per_elem = payload / (tq * d) if tq else 0.0
        return BitReport(payload, params, residual, avg, per_elem, total, tq, tr)
