"""configs[0]-shaped launch (8 units x 4K tokens, G = 4, m4n4, bf16 values; one
layer captured 32 times in a CUDA graph): time per step with the cluster path
(16-CTA clusters when co-schedulable) and without (PQB_DECODE_NO_CLUSTER)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

import os

REPS = int(os.environ.get("PQB_REPS", 32))  # decode calls per captured graph (1: graph launch overhead included)
dev = torch.device("cuda", 0)
w = bench.DecodeWorkload(dev, layers=1, T=4096, batch=1, hq=32, hkv=8, m=4, n=4, page_tokens=256, seed=0)
lib = _lib.load()
res = {"launches": [lib.pqb_decode_launches(w.upl, w.G, w.T, 0), lib.pqb_decode_launches(w.upl, w.G, w.T, _lib.PQB_DECODE_NO_CLUSTER)]}
outs = {}
for rep in range(3):
    for name, fl in (("cluster", 0), ("no_cluster", _lib.PQB_DECODE_NO_CLUSTER)):
        def step(fl=fl):
            for _ in range(REPS):
                w.views[0].decode(w.q[0], out=w.out[0], max_tokens=w.T, flags=fl)
        g = w.capture(step)
        ms = w.timed(g, 10, 3) / REPS
        res.setdefault(name, []).append(round(ms * 1e3, 2))
        g()
        torch.cuda.synchronize()
        outs[name] = w.out.float().clone()
res["max_abs_diff"] = (outs["cluster"] - outs["no_cluster"]).abs().max().item()
print(json.dumps(res))
