"""Summarise one `ncu --set full` capture into a small JSON for profiles/.

usage: python scripts/summarize_ncu.py REPORT.ncu-rep KERNEL_LABEL ALGO_BYTES [OUT.json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_bytes_read": ("dram__bytes_read.sum", None),
    "dram_bytes_write": ("dram__bytes_write.sum", None),
    "dram_throughput_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_active_cycles": ("sm__cycles_active.avg", 1),
    "elapsed_cycles": ("gpc__cycles_elapsed.max", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "lsu_data_pipe_pct": ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1),
    "shared_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    "shared_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "shared_mem_per_block": ("launch__shared_mem_per_block_dynamic", 1),
    "grid_size": ("launch__grid_size", 1),
}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main():
    report, label, algo = sys.argv[1], sys.argv[2], int(sys.argv[3])
    r = raw(report)
    res = {"kernel": label, "source": report.split("/")[-1] + " (ncu --set full --clock-control none, one launch)"}
    for k, (m, scale) in METRICS.items():
        if m in r:
            v, u = r[m]
            x = num(v)
            if x is not None and u in ("MB", "Mbyte") and k.startswith("dram_bytes"):
                x *= 1e6
            elif x is not None and u in ("GB", "Gbyte") and k.startswith("dram_bytes"):
                x *= 1e9
            elif x is not None and u == "KB" and k.startswith("dram_bytes"):
                x *= 1e3
            if x is not None and k == "duration_us":
                x = x / 1e3 if u == "nsecond" else (x if u == "usecond" else x * 1e3 if u == "msecond" else x)
            res[k] = x
    if "dram_bytes_read" in res and "dram_bytes_write" in res:
        res["dram_bytes_per_launch"] = int(res["dram_bytes_read"] + res["dram_bytes_write"])
        res["algorithmic_bytes_per_launch"] = algo
        res["traffic_over_algorithmic"] = round(res["dram_bytes_per_launch"] / algo, 4)
    if "duration_us" in res:
        res["achieved_gbs_under_ncu"] = round(algo / (res["duration_us"] * 1e-6) / 1e9, 1)
    txt = json.dumps(res, indent=1)
    if len(sys.argv) > 4:
        open(sys.argv[4], "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
