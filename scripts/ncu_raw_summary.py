"""Summarise `ncu --page raw --csv` exports (one launch each) into JSON.

    python scripts/ncu_raw_summary.py OUT.json RAW.csv[=ALGO_BYTES] ..."""
import csv
import json
import sys

M = {
    "duration_us": "gpu__time_duration.sum",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "sm_active_cycles": "sm__cycles_active.avg",
    "elapsed_cycles": "gpc__cycles_elapsed.max",
    "sm_clock_ghz": "smsp__cycles_elapsed.avg.per_second",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "shared_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "shared_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "warp_instructions": "smsp__inst_executed.sum",
    "registers_per_thread": "launch__registers_per_thread",
    "grid_size": "launch__grid_size",
}
UNITS = {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}


def summary(path, algo):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    r = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    out = {"kernel": r.get("Kernel Name", ("?", ""))[0], "source": path.split("/")[-1]}
    for k, m in M.items():
        if m not in r:
            continue
        v, u = r[m]
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        if k.startswith("dram_bytes"):
            x *= UNITS.get(u, 1)
        if k == "duration_us":
            x = x / 1e3 if u in ("nsecond", "ns") else x * 1e3 if u in ("msecond", "ms") else x
        out[k] = x
    if "sm_active_cycles" in out and "elapsed_cycles" in out:
        out["sm_active_over_elapsed"] = out["sm_active_cycles"] / out["elapsed_cycles"]
    if algo:
        out["algorithmic_bytes"] = algo
        dram = out.get("dram_bytes_read", 0) + out.get("dram_bytes_write", 0)
        out["dram_bytes"] = dram
        out["traffic_over_algorithmic"] = dram / algo
        out["achieved_gbs_under_ncu"] = algo / (out["duration_us"] * 1e-6) / 1e9
    return out


res = []
for arg in sys.argv[2:]:
    path, _, algo = arg.partition("=")
    res.append(summary(path, int(algo) if algo else None))
json.dump(res, open(sys.argv[1], "w"), indent=1)
print(json.dumps(res, indent=1)[:1500])
