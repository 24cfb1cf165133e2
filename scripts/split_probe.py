"""Per-layer decode time against the persistent grid's CTA count for the
bench shapes (8 layers in a CUDA graph, fused merge policy as shipped):
g4 = configs[1] layer (128 units x 32K), g8 = configs[3] layer (32 x 32K),
m3n2 = configs[2] layer (64 x 128K).  Alternates the CTA counts twice."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

dev = torch.device("cuda", 0)
shapes = {"g4": dict(batch=16, hq=32, hkv=8, m=4, n=4, T=32768), "g8": dict(batch=32, hq=8, hkv=1, m=4, n=4, T=32768),
          "m3n2": dict(batch=8, hq=32, hkv=8, m=3, n=2, T=131072)}
which = sys.argv[1].split(",") if len(sys.argv) > 1 else list(shapes)
res = {}
for name in which:
    kw = shapes[name]
    w = bench.DecodeWorkload(dev, layers=8 if name != "m3n2" else 4, page_tokens=256, seed=0, **kw)
    upl = w.upl
    opts = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "112,120,128,136,140,144,146,148").split(",")]
    for rep in range(3):
        for splits in opts:
            def step(splits=splits):
                for i in range(w.L):
                    w.views[i].decode(w.q[i], out=w.out[i], max_tokens=w.T, splits=splits)
            g = w.capture(step)
            ms = w.timed(g, 8, 3) / w.L
            res.setdefault(f"{name}_{splits}", []).append(round(w.bytes_per_launch() / (ms * 1e-3) / 1e9 / 6546.9, 3))
    w.free()
    del w
    torch.cuda.empty_cache()
print(json.dumps({k: {"median": sorted(v)[len(v) // 2], "reps": v} for k, v in res.items()}))
