"""Can K1 (radius max, memory-bound) and K2 (encode, issue-bound) share the
SMs?  configs[4] slab split in two unit halves: K1(A) alone, K2(B) alone,
then K1(A) on one stream concurrently with K2(B) on another."""
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
cfg = pq.QuantConfig(4, 4)
flags = torch.zeros(1, dtype=torch.int32, device=dev)
ws = torch.empty(U * 64, dtype=torch.int64, device=dev)
cache = pq.PolarKVCache(cfg, U, d, 0, capacity=T, page_tokens=256, value_dtype=torch.bfloat16, device=dev)
h = U // 2
radius_scales_device(keys, cfg, flags, ws, out=cache.scales16)
sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
subB = cache.sub_struct(h, U)
import ctypes


def k1():
    radius_scales_device(keys[:h], cfg, flags, ws[: h * 64], out=cache.scales16[:h])


def k2():
    encode_device(keys[h:], cache.scales16[h:], cfg, ctypes.byref(subB.store), flags=flags)


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


def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    sA.wait_event(ev)
    sB.wait_event(ev)
    with torch.cuda.stream(sA):
        k1()
    with torch.cuda.stream(sB):
        k2()
    cur.wait_stream(sA)
    cur.wait_stream(sB)


res = {"k1_half_ms": timed(k1), "k2_half_ms": timed(k2), "concurrent_ms": timed(both)}
res["sum_ms"] = res["k1_half_ms"] + res["k2_half_ms"]
print(json.dumps({k: round(v, 3) for k, v in res.items()}))
