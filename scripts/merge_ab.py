"""A/B of the split-merge placement (in-kernel vs PQB_DECODE_MERGE_KERNEL) on a
given decode shape: step time per launch, alternating, 3 rounds."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

kw = json.loads(os.environ.get("PQB_SHAPE", '{"batch": 8, "hq": 32, "hkv": 8, "m": 3, "n": 2, "T": 131072}'))
w = bench.DecodeWorkload(torch.device("cuda", 0), layers=8, page_tokens=256, seed=0, **kw)
steps = {f: w.capture(lambda f=f: w.step(f)) for f in (0, _lib.PQB_DECODE_MERGE_KERNEL)}
out = {0: [], 256: []}
for _ in range(3):
    for f, g in steps.items():
        out[f].append(round(w.timed(g, 6, 2) / w.L * 1e3, 2))
print(json.dumps({"shape": kw, "us_per_launch": out}))
