"""Small driver for ncu: a few configs[1]-shaped decode steps (128 units x 32K
tokens per layer, m4n4, G=4); argv[1] = value bits (0: bf16 values, 4: the
4-bit value mode), argv[2] = layers, argv[3] = g4 (default) | g8 (configs[3]
per-GPU launch: 32 units of 8 query heads); page size from PQB_PAGE (256)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench

vb = int(sys.argv[1]) if len(sys.argv) > 1 else 0
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
kind = sys.argv[3] if len(sys.argv) > 3 else "g4"
shape = {"g8": dict(batch=32, hq=8, hkv=1), "m3n2": dict(batch=8, hq=32, hkv=8)}.get(kind, dict(batch=16, hq=32, hkv=8))
m, n, T = (3, 2, 131072) if kind == "m3n2" else (4, 4, 32768)  # m3n2: the configs[2] launch
w = bench.DecodeWorkload(torch.device("cuda", 0), layers=L, T=int(os.environ.get("PQB_T", T)), m=m, n=n,
                         page_tokens=int(os.environ.get("PQB_PAGE", 256)), seed=0, value_bits=vb or None, **shape)
for _ in range(3):
    w.step()
torch.cuda.synchronize()
print("ok")
