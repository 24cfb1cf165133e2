"""Host-side container formats and the synthetic generator (no GPU): PQC1
files and snapshots byte-compatible with the reference (polar_codec.py:367-446,
kv_cache.py:348-397), the reference's error classes, and gen_synthetic_keys
reproducing the reference's PCG64 bytes (tensor_core.py:226-241).  Fixtures:
tests/golden/make_golden_api.py (run against the unmodified reference)."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2502_00527_b200 as pq
from paper_2502_00527_b200 import container

GOLD = Path(__file__).resolve().parent / "golden" / "golden_api.npz"


@pytest.fixture(scope="module")
def gapi():
    data = np.load(GOLD)
    return {k: data[k] for k in data.files}


@pytest.mark.parametrize("i", range(3))
def test_gen_synthetic_keys_matches_reference_bytes(gapi, i):
    T, d, seed, lay = (int(v) for v in gapi[f"syn{i}/meta"])
    cfg = pq.SyntheticConfig(T, d, radius_log_mean=gapi[f"syn{i}/mean"], radius_log_std=gapi[f"syn{i}/std"],
                             outlier_channels=frozenset(gapi[f"syn{i}/outliers"].tolist()),
                             outlier_log_boost=float(gapi[f"syn{i}/boost"]), seed=seed,
                             layout=pq.PairingLayout(lay))
    keys = pq.gen_synthetic_keys(cfg)
    assert keys.data.dtype == np.float32
    assert np.array_equal(keys.data.view(np.uint32), gapi[f"syn{i}/keys"].view(np.uint32))


def test_codes_file_is_byte_compatible(gapi, tmp_path):
    blob = gapi["pqc/blob"].tobytes()
    src = tmp_path / "ref.pqc"
    src.write_bytes(blob)
    codes, scales = pq.load_codes(src)
    dst = tmp_path / "ours.pqc"
    pq.save_codes(codes, scales, dst)
    assert dst.read_bytes() == blob
    assert blob[:4] == pq.CODES_MAGIC


def test_codes_file_errors(gapi, tmp_path):
    good = gapi["pqc/blob"].tobytes()
    p = tmp_path / "c.pqc"
    p.write_bytes(b"NOPE" + good[4:])
    with pytest.raises(pq.BadMagicError):
        pq.load_codes(p)
    p.write_bytes(good[:-2])
    with pytest.raises(pq.TruncatedFileError):
        pq.load_codes(p)
    p.write_bytes(good + b"\x01")
    with pytest.raises(pq.PayloadMismatchError):
        pq.load_codes(p)
    p.write_bytes(good[:3])
    with pytest.raises(pq.TruncatedFileError):
        pq.load_codes(p)
    bad_layout = bytearray(good)
    bad_layout[4 + 10] = 7
    p.write_bytes(bytes(bad_layout))
    with pytest.raises(pq.FormatError):
        pq.load_codes(p)


def test_snapshot_bytes_round_trip(gapi, tmp_path):
    blob = gapi["snap/blob"].tobytes()
    snap = container.parse_snapshot(blob)
    assert container.snapshot_bytes(snap) == blob
    assert snap.residual_keys.shape == (4, 16) and snap.residual_len == 4
    with pytest.raises(pq.TruncatedFileError):
        container.parse_snapshot(blob[:-4])
    with pytest.raises(pq.PayloadMismatchError):
        container.parse_snapshot(blob + b"\0")


@settings(max_examples=30, deadline=None)
@given(tokens=st.integers(0, 40), half=st.integers(1, 12), m=st.integers(1, 8), n=st.integers(1, 8),
       layout=st.sampled_from(list(pq.PairingLayout)), seed=st.integers(0, 2**31 - 1))
def test_codes_file_round_trip(tokens, half, m, n, layout, seed):
    """test_polar_codec.py:296-307 on the host containers."""
    import tempfile

    rng = np.random.default_rng(seed)
    d = 2 * half
    cfg = pq.QuantConfig(m, n, layout)
    a = rng.integers(0, 2**m, tokens * half).astype(np.uint8)
    r = rng.integers(0, 2**n, tokens * half).astype(np.uint8)
    from oracle import polar_oracle as po  # packing oracle (test infrastructure)

    codes = pq.PolarCodes(tokens, d, m, n, layout, po.pack(a, m), po.pack(r, n))
    scales = pq.ChannelScales(rng.uniform(0, 3, half).astype(np.float32))
    with tempfile.TemporaryDirectory() as tmp:
        p = Path(tmp) / "c.pqc"
        pq.save_codes(codes, scales, p)
        c2, s2 = pq.load_codes(p)
    assert c2 == codes and c2.config() == cfg
    assert s2.values.tobytes() == scales.values.tobytes()
