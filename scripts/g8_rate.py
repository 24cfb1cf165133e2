"""configs[3]-shaped layers (32 units x 32K, G = 8, m4n4, bf16 values; 8 layers
in a CUDA graph) with the default launch: per-layer step fraction of the copy
peak (3 reps) and the outputs saved for a cross-build comparison (A/B of
library builds via PQB_LIB; argv[1] = tag)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench

dev = torch.device("cuda", 0)
w = bench.DecodeWorkload(dev, layers=8, T=32768, batch=32, hq=8, hkv=1, m=4, n=4, page_tokens=256, seed=0)
g = w.capture(w.step)
fr = []
for rep in range(3):
    ms = w.timed(g, 8, 3) / w.L
    fr.append(round(w.bytes_per_launch() / (ms * 1e-3) / 1e9 / 6546.9, 3))
g()
torch.cuda.synchronize()
tag = sys.argv[1] if len(sys.argv) > 1 else "x"
Path("gpurun_out").mkdir(exist_ok=True)
torch.save(w.out.float().cpu(), f"gpurun_out/g8_out_{tag}.pt")
print(json.dumps({"tag": tag, "step_frac": fr}))
