"""Top SASS instructions by warp-stall samples from an `ncu --page source
--print-source sass --csv` export (gz ok): python scripts/sass_hot.py FILE [N]."""
import csv, gzip, io, sys
f = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
op = gzip.open if f.endswith(".gz") else open
rows = list(csv.reader(io.TextIOWrapper(op(f, "rb"), encoding="utf-8")))
hdr = rows[1]
ia, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
body = [(i, r) for i, r in enumerate(rows[2:]) if len(r) > ie]
tot = sum(int(r[ia] or 0) for _, r in body)
ins = sum(int(r[ie] or 0) for _, r in body)
print(f"{len(body)} instructions, {tot} samples, {ins} warp-instructions executed")
for i, r in sorted(body, key=lambda x: -int(x[1][ia] or 0))[:n]:
    print(f"{i:5d} {int(r[ia]):7d} {100*int(r[ia])/tot:5.1f}% exec={r[ie]:>9} {r[1].strip()[:90]}")
