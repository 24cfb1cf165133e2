"""Per-SM decode rate: is the spread of CTA loop times across a DQ launch tied
to the SM (systematic) or random?  Runs the trace probe's launch several times
and correlates each SM's tile-loop rate between runs.  Needs a PQB_DQ_TRACE=1
build (PQB_LIB)."""
import ctypes
import json
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
step = w.capture(w.step)
w.timed(step, 10, 3)
lib = _lib.load()
lib.pqb_debug_dq_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
n = torch.cuda.get_device_properties(0).multi_processor_count
rates = []
for rep in range(6):
    buf = np.zeros((n, 32), dtype=np.uint64)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    assert lib.pqb_debug_dq_trace(buf.ctypes.data, n) == 0
    t = buf.astype(np.int64)
    smid = t[:, 30]
    one = t[:, 6] == 0  # single-segment CTAs
    loop_us = (t[:, 3] - t[:, 2]) / 1e3
    tiles = t[:, 29]
    r = np.full(n, np.nan)
    for c in range(n):
        if one[c] and tiles[c] > 0:
            r[smid[c]] = tiles[c] / loop_us[c]  # tiles per us
    rates.append(r)
R = np.array(rates)
ok = ~np.isnan(R).any(axis=0)
Rm = R[:, ok]
corr = np.corrcoef(Rm)
mean = Rm.mean(axis=0)
res = {"shape": shape, "sms_used": int(ok.sum()),
       "rate_tiles_per_us_pct": {p: round(float(np.percentile(mean, p)), 3) for p in (0, 5, 25, 50, 75, 95, 100)},
       "run_to_run_corr_mean": round(float(corr[np.triu_indices(len(rates), 1)].mean()), 3),
       "rel_spread_per_run": [round(float(np.std(x) / np.mean(x)), 4) for x in Rm],
       "rel_spread_of_mean": round(float(np.std(mean) / np.mean(mean)), 4),
       "rate_by_smid": [None if np.isnan(x) else round(float(x), 3) for x in np.nanmean(R, axis=0)]}
print(json.dumps(res))
