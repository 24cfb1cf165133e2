"""Does the per-launch rate depend on the total cache footprint?  Same
configs[1] per-layer launch, caches of L = 4 / 16 / 32 layers."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench

dev = torch.device("cuda", 0)
res = {}
for L in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4,32").split(",")]:
    w = bench.DecodeWorkload(dev, layers=L, batch=16, hq=32, hkv=8, T=32768, m=4, n=4,
                             page_tokens=int(sys.argv[2]) if len(sys.argv) > 2 else 128, seed=0)
    r = bench.measure_workload(w, 20, 5)
    res[f"L{L}"] = {k: round(v, 4) for k, v in r.items()}
    # only the first 4 layers of the big cache
    if L > 4:
        w.L = 4
        r = bench.measure_workload(w, 20, 5)
        res[f"L{L}_first4"] = {k: round(v, 4) for k, v in r.items()}
    del w
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
