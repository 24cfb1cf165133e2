"""Per-launch time of the configs[3]-shaped G=8 decode (32 units of 8 query
heads) against context length: the intercept of time = a + b*T is the fixed
per-launch cost (fill, segment setup, merge tail)."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

dev = torch.device("cuda", 0)
res = {}
for T in [int(t) for t in os.environ.get("PQB_TS", "4096,8192,16384,32768,65536").split(",")]:
    w = bench.DecodeWorkload(dev, layers=8, T=T, batch=32, hq=8, hkv=1, m=4, n=4,
                             page_tokens=int(os.environ.get("PQB_PAGE", 256)), seed=0)
    w.base_flags = int(os.environ.get("PQB_EXTRA_FLAGS", 0))  # A/B of launch variants
    run = w.capture(lambda: w.step(_lib.PQB_DECODE_NO_COMBINE))
    step = w.capture(w.step)
    k = w.timed(run, 6, 2) / w.L
    st = w.timed(step, 6, 2) / w.L
    res[T] = {"kernel_us": round(k * 1e3, 2), "step_us": round(st * 1e3, 2),
              "frac": round(w.bytes_per_launch() / (st * 1e-3) / 1e9 / 6546.9, 3)}
    w.free()
    del w
    torch.cuda.empty_cache()
print(json.dumps(res))
