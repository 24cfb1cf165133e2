"""configs[4] slab (256 units x 131072 bf16 tokens, m4n4): K1 + K2 run
sequentially over the whole slab vs. a chunked two-stream pipeline
(K2 of chunk c on stream A while K1 of chunk c+1 runs on stream B), to see
whether the memory-bound K1 hides under the issue-bound K2."""
import ctypes
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2502_00527_b200 as pq
from paper_2502_00527_b200.codec import encode_device, radius_scales_device

U, T, d = 256, 131072, 128
C = int(os.environ.get("PQB_CHUNK", 16))
dev = torch.device("cuda", 0)
keys = pq.synthetic_keys_device(pq.SyntheticConfig(T, d, outlier_channels=frozenset({0, 1})), U,
                                dtype=torch.bfloat16, device=dev, seed=99)
flags = torch.zeros(1, dtype=torch.int32, device=dev)
ws = torch.empty(U * 64, dtype=torch.int64, device=dev)
cfg = pq.QuantConfig(4, 4)
cache = pq.PolarKVCache(cfg, U, d, 0, capacity=T, page_tokens=256, value_dtype=torch.bfloat16, device=dev)
subs = [cache.sub_struct(u0, u0 + C) for u0 in range(0, U, C)]


def k1(c):
    u0 = c * C
    radius_scales_device(keys[u0:u0 + C], cfg, flags, ws[u0 * 64:(u0 + C) * 64], out=cache.scales16[u0:u0 + C])


def k2(c):
    u0 = c * C
    encode_device(keys[u0:u0 + C], cache.scales16[u0:u0 + C], cfg, ctypes.byref(subs[c].store),
                  clamp_counts=cache.clamp_counts[u0:u0 + C], flags=flags)


def seq():
    radius_scales_device(keys, cfg, flags, ws, out=cache.scales16)
    encode_device(keys, cache.scales16, cfg, cache.store_ref(), clamp_counts=cache.clamp_counts, flags=flags)


sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
n = U // C


def pipe():
    cur = torch.cuda.current_stream()
    sA.wait_stream(cur)
    sB.wait_stream(cur)
    ev = [torch.cuda.Event() for _ in range(n)]
    with torch.cuda.stream(sB):
        for c in range(n):
            k1(c)
            ev[c].record(sB)
    with torch.cuda.stream(sA):
        for c in range(n):
            sA.wait_event(ev[c])
            k2(c)
    cur.wait_stream(sA)
    cur.wait_stream(sB)


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


algo = U * (2 * T * d * 2 + T * (d // 2) * 8 // 8 + 128)
out = {}
for name, fn in [("seq", seq), ("pipe", pipe), ("seq2", seq), ("pipe2", pipe)]:
    ms = timed(fn)
    out[name] = {"ms": round(ms, 3), "frac": round(algo / (ms * 1e-3) / 1e9 / 6546.9, 3)}
print(json.dumps({"lib": os.environ.get("PQB_LIB", ""), "chunk": C, **out}))
