"""Small driver for ncu: a few decode steps of one bench workload.

    python scripts/decode_probe.py VALUES LAYERS KIND
VALUES: bf16 | f32 | vq2 | vq4 | vq8; KIND: g4 (configs[1] launch: 128 units x
32K tokens, m4n4, G = 4), g8 (configs[3] per-GPU launch: 32 units of 8 query
heads), m3n2 (configs[2] launch: 64 units x 128K tokens).  Page size from
PQB_PAGE (256), context from PQB_T."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench

vals = sys.argv[1] if len(sys.argv) > 1 else "bf16"
vals = {"0": "bf16", "4": "vq4"}.get(vals, vals)
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
kind = sys.argv[3] if len(sys.argv) > 3 else "g4"
shape = {"g8": dict(batch=32, hq=8, hkv=1), "m3n2": dict(batch=8, hq=32, hkv=8)}.get(kind, dict(batch=16, hq=32, hkv=8))
m, n, T = (3, 2, 131072) if kind == "m3n2" else (4, 4, 32768)  # m3n2: the configs[2] launch
w = bench.DecodeWorkload(torch.device("cuda", 0), layers=L, T=int(os.environ.get("PQB_T", T)), m=m, n=n,
                         page_tokens=int(os.environ.get("PQB_PAGE", 256)), seed=0, values=vals, **shape)
for _ in range(3):
    w.step()
torch.cuda.synchronize()
print("ok")
