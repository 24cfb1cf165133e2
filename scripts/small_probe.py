"""configs[0]-sized launch (8 units x 4096 tokens, G=4): per-launch time vs CTA count."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench

dev = torch.device("cuda", 0)
w = bench.DecodeWorkload(dev, layers=8, batch=1, hq=32, hkv=8, T=4096, m=4, n=4, page_tokens=128, seed=0)
res = {}
for ctas in [0, 16, 32, 48, 64, 96, 128]:
    def step(c=ctas):
        for i in range(w.L):
            w.views[i].decode(w.q[i], out=w.out[i], max_tokens=w.T, splits=c)
    run = w.capture(step)
    res[ctas] = round(w.timed(run, 20, 3) / w.L * 1e3, 2)
print(json.dumps({"us_per_launch_by_ctas": res}))
