"""configs[3]-shaped layer (32 units x 32K, G = 8, m4n4, bf16 values; 8 layers in
a CUDA graph): per-layer time with the thread-block-cluster DSMEM merge (the
default for this shape) and without it (PQB_DECODE_NO_CLUSTER: balanced split
+ separate merge launch), alternating, plus the outputs' agreement."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

dev = torch.device("cuda", 0)
w = bench.DecodeWorkload(dev, layers=8, T=32768, batch=32, hq=8, hkv=1, m=4, n=4, page_tokens=256, seed=0)
lib = _lib.load()
print("launches per layer:", lib.pqb_decode_launches(w.upl, w.G, w.T, 0), lib.pqb_decode_launches(w.upl, w.G, w.T, _lib.PQB_DECODE_NO_CLUSTER))
res = {"cluster": [], "no_cluster": []}
outs = {}
for rep in range(3):
    for name, fl in (("cluster", 0), ("no_cluster", _lib.PQB_DECODE_NO_CLUSTER)):
        def step(fl=fl):
            for i in range(w.L):
                w.views[i].decode(w.q[i], out=w.out[i], max_tokens=w.T, flags=fl)
        g = w.capture(step)
        ms = w.timed(g, 8, 3) / w.L
        res[name].append(round(w.bytes_per_launch() / (ms * 1e-3) / 1e9 / 6546.9, 3))
        g()
        torch.cuda.synchronize()
        outs[name] = w.out.float().clone()
diff = (outs["cluster"] - outs["no_cluster"]).abs().max().item()
print(json.dumps({"step_frac": res, "max_abs_diff_bf16_out": diff}))
