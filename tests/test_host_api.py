"""Host-side API surface without a GPU: value types mirror the reference's
validation, and every compute entry point fails loudly (no CPU fallback)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2502_00527_b200 as pq
from paper_2502_00527_b200 import core

needs_no_gpu = pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")


def test_public_names_match_reference_boundary():
    for name in ["QuantConfig", "ChannelScales", "PolarCodes", "PairingLayout", "KeyTensor", "PackedKVCache",
                 "compute_radius_scales", "encode_keys", "decode_keys", "build_angle_table", "build_query_lut",
                 "qk_scores", "qk_scores_direct", "attention_weights", "OpCounter", "CacheSnapshot", "BitReport",
                 "FormatError", "BadMagicError", "TruncatedFileError", "PayloadMismatchError", "split_pairs",
                 "merge_pairs", "stream_bytes", "decode_attention", "PolarKVCache"]:
        assert hasattr(pq, name), name


def test_quant_config_validation():
    assert pq.QuantConfig().layout is pq.PairingLayout.HALF_SPLIT
    assert pq.QuantConfig(3, 2).angle_levels == 8 and pq.QuantConfig(3, 2).radius_levels == 4
    for bad in [(0, 4), (4, 9), (9, 1)]:
        with pytest.raises(ValueError):
            pq.QuantConfig(*bad)


def test_layout_values_match_reference_and_abi():
    assert pq.PairingLayout.ADJACENT.value == 0 and pq.PairingLayout.HALF_SPLIT.value == 1
    from paper_2502_00527_b200 import _lib  # noqa: F401  (header: PQB_ADJACENT 0, PQB_HALF_SPLIT 1)


def test_channel_scales():
    s = pq.ChannelScales(np.array([1.0, 0.5]))
    assert s.values.dtype == np.float16 and s.num_channels == 2
    assert s.as_compute().dtype == np.float32
    assert not hasattr(s, "zero_point")
    with pytest.raises(ValueError):
        pq.ChannelScales(np.array([-1.0]))
    with pytest.raises(ValueError):
        pq.ChannelScales(np.array([1e6]))  # fp16 overflow -> inf
    with pytest.raises(ValueError):
        pq.ChannelScales(np.ones((2, 2)))


def test_polar_codes_validation():
    cfg = pq.QuantConfig(4, 4)
    c = pq.PolarCodes(2, 8, 4, 4, cfg.layout, b"\x00" * 4, b"\x00" * 4)
    assert c.config() == cfg
    with pytest.raises(ValueError):
        pq.PolarCodes(2, 8, 4, 4, cfg.layout, b"\x00" * 3, b"\x00" * 4)
    with pytest.raises(ValueError):
        pq.PolarCodes(2, 7, 4, 4, cfg.layout, b"", b"")
    assert pq.stream_bytes(256 * 64, 4) == 256 * 64 * 4 // 8
    assert pq.stream_bytes(5, 3) == 2


def test_pairs_and_key_tensor():
    m = np.arange(8, dtype=np.float32).reshape(1, 8)
    x, y = pq.split_pairs(m, pq.PairingLayout.ADJACENT)
    assert x.tolist() == [[0, 2, 4, 6]] and y.tolist() == [[1, 3, 5, 7]]
    x, y = pq.split_pairs(m, pq.PairingLayout.HALF_SPLIT)
    assert x.tolist() == [[0, 1, 2, 3]]
    assert np.array_equal(pq.merge_pairs(x, y, pq.PairingLayout.HALF_SPLIT), m)
    with pytest.raises(ValueError):
        pq.split_pairs(np.zeros((1, 7)), pq.PairingLayout.ADJACENT)
    kt = pq.KeyTensor(np.zeros((0, 4)))
    assert kt.num_tokens == 0 and kt.dim == 4
    with pytest.raises(ValueError):
        pq.KeyTensor(np.zeros((2, 3)))


def test_op_counter_and_bit_report():
    c = pq.OpCounter(multiplies=5, additions=2, lookups=9)
    c.reset()
    assert c.as_dict() == {"multiplies": 0, "additions": 0, "lookups": 0}
    r = core.BitReport(10, 2, 3, 1.0, 0.5, 4, 3, 1)
    assert r.total_bits == 15 and r.as_dict()["total_bits"] == 15


def test_empty_cache_report_without_gpu():
    cache = pq.PackedKVCache(pq.QuantConfig(4, 4), 0)
    rep = cache.memory_report()
    assert rep.total_bits == 0 and rep.avg_bits_per_element == 0.0
    assert not cache.prefilled and cache.num_tokens == 0
    with pytest.raises(RuntimeError):
        _ = cache.dim
    with pytest.raises(ValueError):
        pq.PackedKVCache(pq.QuantConfig(4, 4), -1)


@needs_no_gpu
@pytest.mark.parametrize(
    "fn",
    [
        lambda: pq.compute_radius_scales(np.ones((4, 8), np.float32), pq.QuantConfig()),
        lambda: pq.encode_keys(np.ones((4, 8), np.float32), pq.ChannelScales(np.ones(4)), pq.QuantConfig()),
        lambda: pq.build_angle_table(4),
        lambda: pq.attention_weights(np.ones(3), 1.0),
        lambda: pq.PackedKVCache(pq.QuantConfig(), 0).prefill(np.ones((4, 8), np.float32)),
        lambda: pq.PolarKVCache(pq.QuantConfig(), 2, 128),
    ],
)
def test_product_fails_loudly_without_gpu(fn):
    with pytest.raises(RuntimeError, match="CUDA"):
        fn()


def test_product_never_imports_oracle():
    import pathlib

    pkg = pathlib.Path(pq.__file__).parent
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f


def test_value_bits_validation_without_gpu():
    """The batched cache's value-quantization mode checks its arguments before
    it touches a device (same ValueError as quantize_uniform's bit check)."""
    import pytest

    import paper_2502_00527_b200 as pq

    with pytest.raises(ValueError):
        pq.PolarKVCache(pq.QuantConfig(4, 4), 1, 128, 0, value_bits=9)
    with pytest.raises(ValueError):
        pq.PolarKVCache(pq.QuantConfig(4, 4), 1, 128, 0, value_bits=3)
    with pytest.raises(ValueError):
        pq.PolarKVCache(pq.QuantConfig(4, 4), 1, 64, 0, value_bits=4)
