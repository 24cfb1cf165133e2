"""Scores-only DQ mode rate (configs[1] shape, 8 layers in a CUDA graph):
fraction of the copy peak over the code bytes; for A/B of
library builds (PQB_LIB)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

dev = torch.device("cuda", 0)
w = bench.DecodeWorkload(dev, layers=8, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, page_tokens=256, seed=7)
sc = torch.empty((w.upl, w.G, w.T), dtype=torch.float32, device=dev)
codes = w.L * w.upl * (w.T * 64 * 8 // 8)


def step():
    for i in range(w.L):
        w.views[i].scores(w.q[i], max_tokens=w.T, out=sc, flags=_lib.PQB_DECODE_DQ)


g = w.capture(step)
ms = w.timed(g, 6, 2)
print(json.dumps({"scores_dq_frac_codes": round(codes / (ms * 1e-3) / 1e9 / 6546.9, 3)}))
