"""LUT vs dequant/tensor-core scoring on the bench shapes (G = 4: configs[1]
per-layer launch; G = 8: configs[3] per-GPU slice), fewer layers."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

dev = torch.device("cuda", 0)
res = {}
variants = sys.argv[1].split(",") if len(sys.argv) > 1 else ["lut", "dq"]
shapes = [("G4_cfg1", dict(batch=16, hq=32, hkv=8)), ("G8_cfg3", dict(batch=32, hq=8, hkv=1))]
if len(sys.argv) > 2:
    shapes = [s for s in shapes if s[0] in sys.argv[2].split(",")]
for name, kw in shapes:
    w = bench.DecodeWorkload(dev, layers=4, T=32768, m=4, n=4, page_tokens=128, seed=0, **kw)
    outs = {}
    for tag, fl in [(v, {"lut": _lib.PQB_DECODE_LUT, "dq": _lib.PQB_DECODE_DQ}[v]) for v in variants]:
        w.base_flags = fl
        r = bench.measure_workload(w, 20, 5)
        w.step()
        torch.cuda.synchronize()
        outs[tag] = w.out.float().clone()
        res[f"{name}_{tag}"] = {k: round(v, 4) for k, v in r.items()}
    if len(outs) == 2:
        res[f"{name}_maxdiff_lut_vs_dq"] = (outs["lut"] - outs["dq"]).abs().max().item()
    del w
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
