"""Burst per-launch rate (fraction of the measured copy peak) of the fused
decode for three shapes, 8-layer caches, short timed runs; for A/B of library
builds (PQB_LIB=...) with cool-down between processes."""
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
for name, kw in [("g4", dict(batch=16, hq=32, hkv=8, m=4, n=4)), ("g8", dict(batch=32, hq=8, hkv=1, m=4, n=4)),
                 ("vq4", dict(batch=16, hq=32, hkv=8, m=4, n=4, values="vq4")),
                 ("m3n2", dict(batch=8, hq=32, hkv=8, m=3, n=2))]:
    T = 131072 if name == "m3n2" else 32768
    w = bench.DecodeWorkload(dev, layers=8, T=T, page_tokens=int(os.environ.get("PQB_PAGE", 128)), seed=0, **kw)
    w.base_flags = int(os.environ.get("PQB_EXTRA_FLAGS", 0))  # A/B of launch variants
    run = w.capture(lambda: w.step(_lib.PQB_DECODE_NO_COMBINE))
    step = w.capture(w.step)
    a = w.bytes_per_launch()
    k = w.timed(run, 6, 2) / w.L
    st = w.timed(step, 6, 2) / w.L
    res[name] = (round(a / (k * 1e-3) / 1e9 / 6546.9, 3), round(a / (st * 1e-3) / 1e9 / 6546.9, 3))
    w.free()
    del w
    torch.cuda.empty_cache()
print(json.dumps(res))
