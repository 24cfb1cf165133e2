"""PQC1 code files and cache snapshots (the reference's on-disk formats).

  save_codes / load_codes        polar_codec.py:367-446
  save_snapshot / load_snapshot  kv_cache.py:348-397

The byte layouts are the reference's, so files written by either package load
in the other.  Parsing and writing are host byte work (headers, offsets,
error classes); the device side of a load is the page scatter of the two
streams into a paged GPU cache (pqb_import_streams), after which the cache
keeps streaming: ``load_snapshot(path).append(...)`` encodes new tokens with
the restored scales, exactly like the reference's restored cache.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .core import (
    BadMagicError,
    CacheSnapshot,
    ChannelScales,
    FormatError,
    PairingLayout,
    PayloadMismatchError,
    PolarCodes,
    TruncatedFileError,
    _MAX_BITS,
    stream_bytes,
)

CODES_MAGIC = b"PQC1"  # polar_codec.py:35
_HEADER = "<IIBBB"  # num_tokens, dim, angle_bits, radius_bits, layout tag
_TAIL = "<III"  # residual_len, resident count, clamp events (kv_cache.py:353-357)


def _codes_blob(codes: PolarCodes, scales: ChannelScales) -> bytes:
    header = CODES_MAGIC + struct.pack(_HEADER, codes.num_tokens, codes.dim, codes.angle_bits, codes.radius_bits,
                                       codes.layout.value)
    return b"".join((header, scales.values.astype("<f2").tobytes(), codes.angle_stream, codes.radius_stream))


def save_codes(codes: PolarCodes, scales: ChannelScales, path: str | Path) -> None:
    """Write codes and scales in the PQC1 container format."""
    if scales.num_channels != codes.dim // 2:
        raise ValueError(f"{scales.num_channels} scales for {codes.dim} dims")
    Path(path).write_bytes(_codes_blob(codes, scales))


def _parse_codes_blob(blob: bytes, origin: str) -> tuple[PolarCodes, ChannelScales, int]:
    """One PQC1 block of ``blob`` and its end offset (polar_codec.py:405-446)."""
    if len(blob) < 4:
        raise TruncatedFileError(f"{origin}: file shorter than the magic")
    if blob[:4] != CODES_MAGIC:
        raise BadMagicError(f"{origin}: expected magic {CODES_MAGIC!r}, got {blob[:4]!r}")
    header_len = 4 + struct.calcsize(_HEADER)
    if len(blob) < header_len:
        raise TruncatedFileError(f"{origin}: header truncated")
    num_tokens, dim, angle_bits, radius_bits, layout_tag = struct.unpack_from(_HEADER, blob, 4)
    try:
        layout = PairingLayout(layout_tag)
    except ValueError as exc:
        raise FormatError(f"{origin}: unknown layout tag {layout_tag}") from exc
    if dim < 2 or dim % 2:
        raise FormatError(f"{origin}: invalid dim {dim}")
    if not (1 <= angle_bits <= _MAX_BITS and 1 <= radius_bits <= _MAX_BITS):
        raise FormatError(f"{origin}: bit widths ({angle_bits}, {radius_bits}) out of range")
    half = dim // 2
    count = num_tokens * half
    offset = header_len
    bounds = []
    for name, size in (("scales", 2 * half), ("angle stream", stream_bytes(count, angle_bits)),
                       ("radius stream", stream_bytes(count, radius_bits))):
        if len(blob) < offset + size:
            raise TruncatedFileError(f"{origin}: {name} truncated")
        bounds.append((offset, offset + size))
        offset += size
    scales = ChannelScales(np.frombuffer(blob[bounds[0][0]:bounds[0][1]], dtype="<f2"))
    codes = PolarCodes(num_tokens=num_tokens, dim=dim, angle_bits=angle_bits, radius_bits=radius_bits, layout=layout,
                       angle_stream=blob[bounds[1][0]:bounds[1][1]], radius_stream=blob[bounds[2][0]:bounds[2][1]])
    return codes, scales, offset


def load_codes(path: str | Path) -> tuple[PolarCodes, ChannelScales]:
    """Read a PQC1 file; the inverse of :func:`save_codes`.  Bad magic,
    truncation and trailing bytes raise their own FormatError subclasses."""
    blob = Path(path).read_bytes()
    codes, scales, offset = _parse_codes_blob(blob, str(path))
    if offset != len(blob):
        raise PayloadMismatchError(f"{path}: {len(blob) - offset} trailing bytes beyond the code streams")
    return codes, scales


def snapshot_bytes(snap: CacheSnapshot) -> bytes:
    """A PQC1 block plus the residual section (kv_cache.py:348-360)."""
    residual = np.asarray(snap.residual_keys, dtype="<f4")
    return b"".join((_codes_blob(snap.codes, snap.scales),
                     struct.pack(_TAIL, snap.residual_len, residual.shape[0], snap.clamp_events),
                     residual.tobytes()))


def save_snapshot(cache, path: str | Path) -> None:
    """Serialize ``cache.snapshot()``: codes, scales, residual keys (oldest
    first) and the clamp counter.  Values are not serialized."""
    Path(path).write_bytes(snapshot_bytes(cache.snapshot()))


def parse_snapshot(blob: bytes, origin: str = "<bytes>") -> CacheSnapshot:
    """Decode a snapshot file (kv_cache.py:369-385) without building a cache."""
    codes, scales, offset = _parse_codes_blob(blob, origin)
    tail = struct.calcsize(_TAIL)
    if len(blob) < offset + tail:
        raise TruncatedFileError(f"{origin}: residual section header truncated")
    residual_len, count, clamp_events = struct.unpack_from(_TAIL, blob, offset)
    offset += tail
    expected = count * codes.dim * 4
    if len(blob) < offset + expected:
        raise TruncatedFileError(f"{origin}: residual keys truncated")
    if len(blob) > offset + expected:
        raise PayloadMismatchError(f"{origin}: {len(blob) - offset - expected} trailing bytes beyond the residual keys")
    residual = np.frombuffer(blob, dtype="<f4", count=count * codes.dim, offset=offset)
    residual = residual.reshape(count, codes.dim).astype(np.float32)
    return CacheSnapshot(codes=codes, scales=scales, residual_keys=residual, residual_len=residual_len,
                         clamp_events=clamp_events)


def load_snapshot(path: str | Path, device=None):
    """Rebuild a prefilled PackedKVCache on the GPU from :func:`save_snapshot`
    output (kv_cache.py:363-397).  The returned cache accepts further appends;
    stored values come back as zeros (the format carries keys only)."""
    from .cache import PackedKVCache

    snap = parse_snapshot(Path(path).read_bytes(), str(path))
    return PackedKVCache.from_snapshot(snap, device=device)


__all__ = ["CODES_MAGIC", "save_codes", "load_codes", "save_snapshot", "load_snapshot", "parse_snapshot",
           "snapshot_bytes"]
