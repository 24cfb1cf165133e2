"""SASS evidence for profiles/: opcode histogram of one kernel of
libpqb200.so plus the instructions proving the data movement / math units
(UBLKCP = cp.async.bulk TMA copy, SYNCS = mbarrier, LDSM = ldmatrix,
HMMA = mma.sync tensor-core MMA, PRMT / LDS gather).

    python scripts/sass_excerpt.py MANGLED_NAME_SUBSTRING OUT.txt"""
import collections
import re
import subprocess
import sys
from pathlib import Path

lib = Path(__file__).resolve().parents[1] / "paper_2502_00527_b200" / "libpqb200.so"
pat, out = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
body = next(f for f in funcs if f.split("\n", 1)[0].strip().find(pat) >= 0)
name = body.split("\n", 1)[0].strip()
ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+([^;]*);", body)
ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", i).split()[0] for i in ins)
keys = ("UBLKCP", "SYNCS", "LDSM", "HMMA", "PRMT", "LDS", "MUFU", "SHFL", "STG", "REDG", "BAR", "UTC", "LDTM")
with open(out, "w") as fh:
    fh.write(f"kernel: {name}\nsource: cuobjdump -sass {lib.name} (sm_100a)\n{len(ins)} instructions\n\n")
    fh.write("opcode histogram (top 40):\n")
    for op, c in ops.most_common(40):
        fh.write(f"  {op:28s} {c}\n")
    fh.write("\nkey instruction families:\n")
    for k in keys:
        fam = {op: c for op, c in ops.items() if op.startswith(k)}
        if fam:
            fh.write(f"  {k}: {fam}\n")
    fh.write("\nfirst occurrences:\n")
    seen = set()
    for i in ins:
        op = re.sub(r"^@!?U?P\w+\s+", "", i).split()[0]
        fam = next((k for k in keys if op.startswith(k)), None)
        if fam and op not in seen:
            seen.add(op)
            fh.write(f"  {i.strip()}\n")
print(out)
