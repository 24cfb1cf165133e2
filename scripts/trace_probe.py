"""Launch-phase trace of one DQ decode launch (needs a PQB_DQ_TRACE=1 build):

    PQB_LIB=build_ab/libpqb200_trace.so python scripts/trace_probe.py [g8|g4]

Runs the configs[3]- (g8: 32 units of 8 query heads, 32K) or configs[1]-shaped
(g4: 128 units of 4, 32K) decode step in a CUDA graph (8 layers, PDL between
launches) and reads back the %globaltimer stamps of the last layer's launch:
per CTA entry, grid-dependency wait, per segment setup / tile loop / epilogue,
exit.  Prints a JSON summary of where the launch time goes."""
import ctypes
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2502_00527_b200 import _lib

shape = sys.argv[1] if len(sys.argv) > 1 else "g8"
dev = torch.device("cuda", 0)
if shape == "g8":
    w = bench.DecodeWorkload(dev, layers=8, T=32768, batch=32, hq=8, hkv=1, m=4, n=4, page_tokens=256, seed=0)
else:
    w = bench.DecodeWorkload(dev, layers=8, T=32768, batch=16, hq=32, hkv=8, m=4, n=4, page_tokens=256, seed=0)
w.base_flags = int(os.environ.get("PQB_EXTRA_FLAGS", 0))
step = w.capture(w.step)
ms = w.timed(step, 10, 3) / w.L
lib = _lib.load()
lib.pqb_debug_dq_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
n = torch.cuda.get_device_properties(0).multi_processor_count
buf = np.zeros((n, 32), dtype=np.uint64)
step()
torch.cuda.synchronize()
assert lib.pqb_debug_dq_trace(buf.ctypes.data, n) == 0
t = buf.astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3  # us
segs = []
for c in range(n):
    k = 0
    while k < 6 and t[c, 2 + 4 * k] != 0 and t[c, 4 + 4 * k] >= t[c, 2 + 4 * k]:
        prev = t[c, 1] if k == 0 else t[c, 4 + 4 * (k - 1)]
        segs.append({"cta": c, "k": k, "unit": int(t[c, 5 + 4 * k]),
                     "setup_us": (t[c, 2 + 4 * k] - prev) / 1e3,
                     "loop_us": (t[c, 3 + 4 * k] - t[c, 2 + 4 * k]) / 1e3,
                     "epi_us": (t[c, 4 + 4 * k] - t[c, 3 + 4 * k]) / 1e3})
        k += 1
ends = rel[:, 31]
waits = rel[:, 1]
pct = lambda a: {p: round(float(np.percentile(a, p)), 2) for p in (0, 10, 50, 90, 100)}
res = {
    "shape": shape, "layer_us_graph": round(ms * 1e3, 2),
    "entry_us": pct(rel[:, 0]), "wait_done_us": pct(waits), "exit_us": pct(ends),
    "span_us": round(float(ends.max()), 2),
    "segments_per_cta": pct(np.bincount([s["cta"] for s in segs], minlength=n)),
    "setup_us": pct([s["setup_us"] for s in segs]),
    "loop_us": pct([s["loop_us"] for s in segs]),
    "epi_us": pct([s["epi_us"] for s in segs]),
    "epi_first_seg_us": pct([s["epi_us"] for s in segs if s["k"] == 0]),
    "epi_last_seg_us": pct([s["epi_us"] for s in segs if s["k"] > 0]) if any(s["k"] > 0 for s in segs) else None,
}
print(json.dumps(res))
Path("gpurun_out").mkdir(exist_ok=True)
np.save(f"gpurun_out/trace_{shape}.npy", buf)
