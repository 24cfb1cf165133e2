"""Memory-footprint sensitivity: copy bandwidth and the decode launch with and
without 38 GB of other live allocations."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench


def copy_bw(n_bytes=1 << 31, reps=20):
    a = torch.empty(n_bytes // 2, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    del a, b
    return 2 * n_bytes / (ms * 1e-3) / 1e9


dev = torch.device("cuda", 0)
res = {"copy_small_footprint_gbs": copy_bw()}
w = bench.DecodeWorkload(dev, layers=4, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, page_tokens=128, seed=0)
res["dq_L4"] = bench.measure_workload(w, 20, 5)["frac"]
dummy = torch.empty(38 << 30, dtype=torch.uint8, device="cuda")
dummy.fill_(1)
res["copy_with_38GB_live_gbs"] = copy_bw()
res["dq_L4_with_38GB_live"] = bench.measure_workload(w, 20, 5)["frac"]
del dummy
torch.cuda.empty_cache()
res["dq_L4_after_free"] = bench.measure_workload(w, 20, 5)["frac"]
del w
torch.cuda.empty_cache()
big = torch.empty(40 << 30, dtype=torch.uint8, device="cuda")
big.fill_(0)
x = big[: 1 << 31]
y = big[20 << 30: (20 << 30) + (1 << 31)]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    y.copy_(x)
e0.record()
for _ in range(20):
    y.copy_(x)
e1.record()
e1.synchronize()
res["copy_inside_40GB_alloc_gbs"] = 2 * (1 << 31) / (e0.elapsed_time(e1) / 20 * 1e-3) / 1e9
print(json.dumps(res, indent=1))
