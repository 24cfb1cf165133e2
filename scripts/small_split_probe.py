"""configs[0] (1 layer, 8 units x 4K tokens, G=4) launch time against the CTA
count handed to the split (UnitView.decode splits=): where the short-launch
split should land."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench

w = bench.DecodeWorkload(torch.device("cuda", 0), layers=4, batch=1, hq=32, hkv=8, T=4096, m=4, n=4,
                         page_tokens=256, seed=0)
res = {}
for ctas in (0, 16, 32, 48, 64, 96, 128):
    def step(ctas=ctas):
        for i in range(w.L):
            w.views[i].decode(w.q[i], out=w.out[i], max_tokens=w.T, splits=ctas)
    g = w.capture(step)
    res[ctas] = [round(w.timed(g, 50, 5) / w.L * 1e3, 2) for _ in range(2)]
from paper_2502_00527_b200 import _lib


def step_mk():
    for i in range(w.L):
        w.views[i].decode(w.q[i], out=w.out[i], max_tokens=w.T, flags=_lib.PQB_DECODE_MERGE_KERNEL)


g = w.capture(step_mk)
res["default+merge_kernel"] = [round(w.timed(g, 50, 5) / w.L * 1e3, 2) for _ in range(2)]
print(json.dumps({"us_per_launch_by_ctas": res}))
