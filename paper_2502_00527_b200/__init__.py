"""paper_2502_00527_b200 -- B200-native PolarQuant hot path.

Drop-in for the key-cache encoder and LUT decode attention of the PolarQuant
reference (``import polarquant as pq`` -> ``import paper_2502_00527_b200 as pq``).
All arithmetic runs in libpqb200.so (hand-written sm_100a CUDA behind a C ABI,
include/pqb200.h); there is no CPU fallback.
"""

from .attention import (
    attention_weights,
    build_angle_table,
    build_query_lut,
    decode_attention,
    qk_scores,
    qk_scores_direct,
)
from .cache import PackedKVCache, PolarKVCache
from .codec import (
    angle_grid,
    compute_radius_scales,
    decode_keys,
    encode_keys,
    quantize_angle,
    quantize_radius,
    to_polar,
)
from .container import CODES_MAGIC, load_codes, load_snapshot, save_codes, save_snapshot
from .core import (
    AngleTable,
    BadMagicError,
    BitReport,
    CacheSnapshot,
    ChannelScales,
    FormatError,
    KeyTensor,
    OpCounter,
    PairingLayout,
    PayloadMismatchError,
    PolarCodes,
    QuantConfig,
    QueryLUT,
    TruncatedFileError,
    merge_pairs,
    split_pairs,
    stream_bytes,
)
from .synthetic import SyntheticConfig, gen_synthetic_keys, normal_device, synthetic_keys_device

__version__ = "0.1.0"

__all__ = [
    "CODES_MAGIC",
    "AngleTable",
    "BadMagicError",
    "BitReport",
    "CacheSnapshot",
    "ChannelScales",
    "FormatError",
    "KeyTensor",
    "OpCounter",
    "PackedKVCache",
    "PairingLayout",
    "PayloadMismatchError",
    "PolarCodes",
    "PolarKVCache",
    "QuantConfig",
    "QueryLUT",
    "SyntheticConfig",
    "TruncatedFileError",
    "angle_grid",
    "attention_weights",
    "build_angle_table",
    "build_query_lut",
    "compute_radius_scales",
    "decode_attention",
    "decode_keys",
    "encode_keys",
    "gen_synthetic_keys",
    "load_codes",
    "load_snapshot",
    "merge_pairs",
    "normal_device",
    "qk_scores",
    "qk_scores_direct",
    "quantize_angle",
    "quantize_radius",
    "save_codes",
    "save_snapshot",
    "split_pairs",
    "stream_bytes",
    "synthetic_keys_device",
    "to_polar",
]
