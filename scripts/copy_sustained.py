"""HBM copy bandwidth: burst (first reps) vs after seconds of sustained load."""
import json
import time

import torch

n = 1 << 30  # bf16 elements (2 GiB per buffer)
a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
a.fill_(1)


def bw(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    e1.synchronize()
    return round(4 * n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)


res = {"burst_first10": bw(10)}
t0 = time.time()
seq = []
while time.time() - t0 < 6:
    seq.append(bw(50))
res["sustained_series_50reps"] = seq
res["after_6s_10reps"] = bw(10)
time.sleep(3)
res["after_3s_idle_10reps"] = bw(10)
print(json.dumps(res))
