"""Sustained configs[1] decode: per-chunk launch rate for ~4 s of back-to-back
steps, with nvidia-smi sampling SM clock / power / throttle reasons every 50 ms
(written to gpurun_out/sustain_clocks.csv) to tell a power/clock cause from a
memory-system one."""
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
vbits = int(sys.argv[2]) if len(sys.argv) > 2 else None  # 4: the 4-bit value mode
dev = torch.device("cuda", 0)
w = bench.DecodeWorkload(dev, layers=32, batch=16, hq=32, hkv=8, T=32768, m=4, n=4, page_tokens=int(os.environ.get("PQB_PAGE", 256)), seed=0,
                         value_bits=vbits)
algo = w.bytes_per_launch()
spl = int(os.environ.get("PQB_SPLITS", 0))  # CTA count handed to the split (0: one per SM)


def step_s(f):
    for i in range(w.L):
        w.views[i].decode(w.q[i], out=w.out[i], max_tokens=w.T, flags=f, splits=spl)


run = w.capture(lambda: step_s(_lib.PQB_DECODE_NO_COMBINE | flags))
Path("gpurun_out").mkdir(exist_ok=True)
smi = subprocess.Popen(
    ["nvidia-smi", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,"
     "clocks_event_reasons.active", "--format=csv", "-lms", "50"],
    stdout=open("gpurun_out/sustain_clocks.csv", "w"), stderr=subprocess.DEVNULL)
time.sleep(1.0)
t0 = time.time()
rates = []
while time.time() - t0 < 4.0:
    ms = w.timed(run, 4, 0) / w.L
    rates.append(round(algo / (ms * 1e-3) / 1e9 / 6546.9, 3))
time.sleep(0.5)
idle_after = []
time.sleep(2.0)
for _ in range(3):
    ms = w.timed(run, 2, 0) / w.L
    idle_after.append(round(algo / (ms * 1e-3) / 1e9 / 6546.9, 3))
smi.terminate()
step_ms = w.timed(w.capture(w.step), 10, 2)
print(json.dumps({"flags": flags, "value_bits": vbits, "lib": os.environ.get("PQB_LIB", ""), "splits": spl,
                  "median_last_half": statistics.median(rates[len(rates) // 2:]), "chunk_rates": rates, "after_2s_idle": idle_after,
                  "tokens_per_s_cool": round(w.batch / (step_ms * 1e-3), 1)}))
