"""Where does the configs[1] decode launch spend its time?  Same per-layer
launch (128 units x 32K tokens, m4n4, G=4), three builds of the DQ kernel:
the kernel, memory only (tiles stream, no compute), compute only (tiles from
L2).  Reported as fraction of the measured copy peak (algorithmic bytes), for
a short burst and after a few seconds of sustained decode."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32
G = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dev = torch.device("cuda", 0)
if G == 4:
    w = bench.DecodeWorkload(dev, layers=L, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, page_tokens=128, seed=0)
else:
    w = bench.DecodeWorkload(dev, layers=L, batch=32, hq=8, hkv=1, T=32768, m=4, n=4, page_tokens=128, seed=0)
algo = w.bytes_per_launch()
peak = 6546.9
res = {"layers": L, "G": G}
for name, fl in [("kernel", 0), ("mem_only", _lib.PQB_DECODE_PROBE_MEM), ("compute_only", _lib.PQB_DECODE_PROBE_COMPUTE),
                 ("kernel_again", 0)]:
    run = w.capture(lambda fl=fl: w.step(_lib.PQB_DECODE_NO_COMBINE | fl))
    r = []
    for reps in (3, 3, 30, 30, 3):
        ms = w.timed(run, reps, 1) / w.L
        r.append(round(algo / (ms * 1e-3) / 1e9 / peak, 4))
    res[name] = r
print(json.dumps(res))

# read-only and copy references on a 16 GiB buffer (bytes touched / time)
del w
torch.cuda.empty_cache()
x = torch.ones(1 << 32, dtype=torch.float32, device=dev)
y = torch.empty(1 << 31, dtype=torch.float32, device=dev)


def rate(fn, nbytes, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return round(nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)


res["torch_sum_read_gbs"] = [rate(lambda: x.sum(), x.numel() * 4, r) for r in (5, 40)]
res["torch_copy_gbs"] = [rate(lambda: y.copy_(x[: 1 << 31]), 2 * y.numel() * 4, r) for r in (5, 40)]
print(json.dumps(res))
