"""Summarise a DQ launch-phase trace (scripts/trace_probe.py output):
per-CTA entry / grid-dependency wait / exit, warp 0's run phases."""
import json
import sys

import numpy as np

t = np.load(sys.argv[1]).astype(np.int64)
t0 = t[:, 0].min()
r = (t - t0) / 1e3
pct = lambda a: {p: round(float(np.percentile(a, p)), 2) for p in (0, 10, 50, 90, 100)} if len(a) else None
setup, loop, flush = [], [], []
for c in range(t.shape[0]):
    prev = t[c, 1]
    for k in range(6):
        if t[c, 2 + 4 * k] == 0 or t[c, 4 + 4 * k] < t[c, 2 + 4 * k]:
            break
        setup.append((t[c, 2 + 4 * k] - prev) / 1e3)
        loop.append((t[c, 3 + 4 * k] - t[c, 2 + 4 * k]) / 1e3)
        flush.append((t[c, 4 + 4 * k] - t[c, 3 + 4 * k]) / 1e3)
        prev = t[c, 4 + 4 * k]
last_flush = (t[:, 31] - np.max(np.where(t[:, 4:28:4] > 0, t[:, 4:28:4], 0), axis=1)) / 1e3
print(json.dumps({"entry": pct(r[:, 0]), "wait_done": pct(r[:, 1]), "exit": pct(r[:, 31]),
                  "w0_setup": pct(setup), "w0_loop": pct(loop), "w0_flush": pct(flush),
                  "cta_epilogue_after_w0": pct(last_flush)}))
