"""K1 (scales) and K2 (encode) device times on the configs[4] slab
(256 units x 131072 bf16 tokens), per (m, n); PQB_ENCODE_KERNEL=v8 selects the
per-call-grid encoder for A/B."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2502_00527_b200 as pq
from paper_2502_00527_b200.codec import encode_device, radius_scales_device

U, T, d = 256, 131072, 128
dev = torch.device("cuda", 0)
keys = pq.synthetic_keys_device(pq.SyntheticConfig(T, d, outlier_channels=frozenset({0, 1})), U,
                                dtype=torch.bfloat16, device=dev, seed=99)
flags = torch.zeros(1, dtype=torch.int32, device=dev)
ws = torch.empty(U * 64, dtype=torch.int64, device=dev)
peak = 6546.9


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
for m, n in [(4, 4), (3, 2), (2, 4)]:
    cfg = pq.QuantConfig(m, n)
    cache = pq.PolarKVCache(cfg, U, d, 0, capacity=T, page_tokens=256, value_dtype=torch.bfloat16, device=dev)
    k1 = timed(lambda: radius_scales_device(keys, cfg, flags, ws, out=cache.scales16))
    k2 = timed(lambda: encode_device(keys, cache.scales16, cfg, cache.store_ref(), clamp_counts=cache.clamp_counts,
                                     flags=flags))
    kb = U * T * d * 2
    cb = U * T * 64 * (m + n) // 8
    res[f"m{m}n{n}"] = {"k1_ms": round(k1, 3), "k1_frac": round(kb / (k1 * 1e-3) / 1e9 / peak, 3),
                        "k2_ms": round(k2, 3), "k2_frac": round((kb + cb) / (k2 * 1e-3) / 1e9 / peak, 3),
                        "total_frac": round((2 * kb + cb) / ((k1 + k2) * 1e-3) / 1e9 / peak, 3)}
    del cache
    torch.cuda.empty_cache()
print(json.dumps(res))
