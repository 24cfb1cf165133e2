"""Per-unit parity of the bench's quantized-value extras (diagnostics)."""
import sys, math
import numpy as np, torch
sys.path.insert(0, '.')
import bench
from oracle import parity
from paper_2502_00527_b200 import _lib

vals = sys.argv[1] if len(sys.argv) > 1 else "vq2"
dev = torch.device("cuda", 0)
keep = bench.sample_units(128, 32, 8, 5, all_layer0=False)
w = bench.DecodeWorkload(dev, layers=32, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, page_tokens=256, seed=7,
                         values=vals, keep=keep)
run = w.capture(w.step)
with torch.cuda.stream(w.stream):
    run()
torch.cuda.synchronize()
jobs = w.parity_jobs(keep)
for u, j in zip(keep, jobs):
    r = parity.check_unit(**j)
    layer, jj = divmod(u, w.upl)
    q = w.q[layer, jj:jj + 1]
    o32 = w.views[layer].decode(w.q[layer], out_dtype=torch.float32)[jj].cpu().numpy()
    gen = w.views[layer].decode(w.q[layer], out_dtype=torch.float32, flags=_lib.PQB_DECODE_FORCE_GENERIC)[jj].cpu().numpy()
    v64 = j["values"].astype(np.float64)
    from oracle import exact, polar_oracle as po
    s16 = w.cache.scales16[u].cpu().numpy()
    errs = []
    for g in range(4):
        sc = exact.lut_scores(j["q"][g], j["angle_gpu"], j["radius_gpu"], s16, 4, 4, 1)
        ref = po.softmax64(sc, 1 / math.sqrt(128)) @ v64
        errs.append((float(np.abs(ref).max()), float(np.abs(o32[g] - ref).max()), float(np.abs(gen[g] - ref).max()),
                     float(np.abs(j["out"][g] - ref).max())))
    print(u, r.out_err, r.out_excess, [tuple(round(x, 6) for x in e) for e in errs], flush=True)
