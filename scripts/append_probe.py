"""Streaming append (K5) cost at the configs[1] decode-step shape: one new
token for every unit of a 32-layer, batch-16 cache (4096 units), with and
without a residual window; device time per append call vs the decode step."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2502_00527_b200 as pq

dev = torch.device("cuda", 0)
res = {}
for R, vb in [(0, None), (128, None), (0, 4)]:
    U, T = 4096, 2048
    cache = pq.PolarKVCache(pq.QuantConfig(4, 4), U, 128, R, capacity=T + 64, page_tokens=128, device=dev,
                            value_bits=vb)
    keys = pq.synthetic_keys_device(pq.SyntheticConfig(T, 128), U, dtype=torch.bfloat16, device=dev, seed=1)
    vals = pq.normal_device((U, T, 128), 2, dtype=torch.bfloat16, device=dev)
    cache.prefill(keys, vals)
    del keys, vals
    k = pq.normal_device((U, 128), 3, dtype=torch.bfloat16, device=dev)
    v = pq.normal_device((U, 128), 4, dtype=torch.bfloat16, device=dev)
    for _ in range(3):
        cache.append(k, v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        cache.append(k, v)
    e1.record()
    torch.cuda.synchronize()
    res[f"res{R}_vbits{vb}"] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
    del cache
    torch.cuda.empty_cache()
print(json.dumps({"us_per_append_4096_units": res}))
