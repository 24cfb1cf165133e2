"""Per-launch rate vs length of the timed run (thermal / power / refresh drift)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

dev = torch.device("cuda", 0)
w = bench.DecodeWorkload(dev, layers=4, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, page_tokens=128, seed=0)
run_attn = w.capture(lambda: w.step(_lib.PQB_DECODE_NO_COMBINE))
algo = w.bytes_per_launch()
res = {}
for reps in [10, 50, 250, 1000, 10, 2000, 10]:
    ms = w.timed(run_attn, reps, 2) / w.L
    res.setdefault(str(reps), []).append(round(algo / (ms * 1e-3) / 1e9 / 6547.8, 4))
print(json.dumps(res))
