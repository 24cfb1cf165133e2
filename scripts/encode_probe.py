"""Small driver for ncu: one config-5 style encode (K1 + K2) of 64 units x 64K bf16 tokens."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2502_00527_b200 as pq
from paper_2502_00527_b200.codec import encode_device, radius_scales_device

U, T = 64, 65536
m = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = pq.QuantConfig(m, n)
keys = pq.synthetic_keys_device(pq.SyntheticConfig(T, 128, outlier_channels=frozenset({0, 1})), U)
cache = pq.PolarKVCache(cfg, U, 128, 0, capacity=T, page_tokens=256)
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    radius_scales_device(keys, cfg, flags, out=cache.scales16)
    encode_device(keys, cache.scales16, cfg, cache.store_ref(), clamp_counts=cache.clamp_counts, flags=flags)
torch.cuda.synchronize()
print("ok")
