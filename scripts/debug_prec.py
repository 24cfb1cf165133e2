"""fp32-output precision of the fused decode at the bench's context length,
per value treatment (diagnostics): max |o - ref| / max |ref| over sampled units."""
import sys, math
import numpy as np, torch
sys.path.insert(0, '.')
import bench
from oracle import exact, polar_oracle as po
from paper_2502_00527_b200 import _lib

dev = torch.device("cuda", 0)
T = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
for vals in sys.argv[1].split(","):
    keep = list(range(0, 128, 16))
    w = bench.DecodeWorkload(dev, layers=1, batch=16, hq=32, hkv=8, T=T, m=4, n=4, page_tokens=256, seed=7,
                             values=vals, keep=keep)
    o32 = w.views[0].decode(w.q[0], out_dtype=torch.float32).cpu().numpy()
    gen = w.views[0].decode(w.q[0], out_dtype=torch.float32, flags=_lib.PQB_DECODE_FORCE_GENERIC).cpu().numpy()
    worst, worst_g = 0.0, 0.0
    for u in keep:
        keys, vv = w.kept[u]
        v64 = (w.cache.values_f32(u) if vals.startswith("vq") else vv.float()).cpu().numpy().astype(np.float64)
        a, r = (t.cpu().numpy() for t in w.cache.code_arrays(u))
        s16 = w.cache.scales16[u].cpu().numpy()
        q = w.q[0, u].float().cpu().numpy()
        for g in range(4):
            ref = po.softmax64(exact.lut_scores(q[g], a, r, s16, 4, 4, 1), 1 / math.sqrt(128)) @ v64
            pk = max(1.0, float(np.abs(ref).max()))
            worst = max(worst, float(np.abs(o32[u, g] - ref).max()) / pk)
            worst_g = max(worst_g, float(np.abs(gen[u, g] - ref).max()) / pk)
    print(f"{vals} T={T}: dq max rel err {worst:.3e}   generic {worst_g:.3e}", flush=True)
    w.free()
