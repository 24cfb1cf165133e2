"""configs[3]-shaped G=8 layer (32 units x 32K, m4n4, bf16 values, 8 layers in a
CUDA graph): per-layer time against the persistent grid's CTA count and the
split-merge placement (separate PDL launch vs last CTA in the decode launch)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

dev = torch.device("cuda", 0)
w = bench.DecodeWorkload(dev, layers=8, T=32768, batch=32, hq=8, hkv=1, m=4, n=4, page_tokens=256, seed=0)
res = {}
for splits in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "148,144,140,136,132,128").split(",")]:
    for name, fl in (("sep", 0), ("inkernel", _lib.PQB_DECODE_MERGE_INKERNEL), ("nocombine", _lib.PQB_DECODE_NO_COMBINE)):
        def step(fl=fl, splits=splits):
            for i in range(w.L):
                w.views[i].decode(w.q[i], out=w.out[i], max_tokens=w.T, flags=fl, splits=splits)
        g = w.capture(step)
        ms = w.timed(g, 8, 3) / w.L
        res[f"{splits}_{name}"] = {"layer_us": round(ms * 1e3, 2),
                                   "frac": round(w.bytes_per_launch() / (ms * 1e-3) / 1e9 / 6546.9, 3)}
print(json.dumps(res))
