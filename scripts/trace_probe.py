"""Launch-phase trace of one DQ decode launch (needs a PQB_DQ_TRACE=1 build):

    PQB_LIB=build_ab/libpqb200_trace.so python scripts/trace_probe.py [g8|g4]

Runs the configs[3]- (g8: 32 units of 8 query heads, 32K) or configs[1]-shaped
(g4: 128 units of 4, 32K) decode step in a CUDA graph (8 layers, PDL between
launches) and reads back the %globaltimer stamps of the last layer's launch:
per CTA entry, grid-dependency wait, per run of warp 0 setup / tile loop /
flush, exit, SM id.  Saves the stamps (gpurun_out/trace_<shape>.npy) for
scripts/trace_summary.py."""
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
print(json.dumps({"shape": shape, "layer_us_graph": round(ms * 1e3, 2)}))
Path("gpurun_out").mkdir(exist_ok=True)
np.save(f"gpurun_out/trace_{shape}.npy", buf)
