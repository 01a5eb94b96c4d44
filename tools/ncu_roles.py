"""Per-role (producer / consumer warps) instruction mix and warp-stall
breakdown from an ncu source-page CSV of a warp-specialised kernel (the role
boundary is the consumer's USETMAXREG.TRY_ALLOC, else the producer's EXIT).
usage: ncu -i rep --page source --csv --print-source sass > x.csv;
       python tools/ncu_roles.py x.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ei = h.index("Source"), h.index("Instructions Executed")
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ops = {"P": collections.Counter(), "C": collections.Counter()}
st = {"P": collections.Counter(), "C": collections.Counter()}
region = "P"
has_alloc = any("TRY_ALLOC" in r[si] for r in rows[2:])
for r in rows[2:]:
    src = r[si].strip()
    if region == "P" and (("TRY_ALLOC" in src) if has_alloc else src.startswith("EXIT")):
        region = "C"
    op = re.sub(r"^@!?U?P[0-9T]+\s+", "", src).split(" ")[0].split(".")[0]
    ops[region][op] += int(r[ei] or 0)
    for c in stalls:
        st[region][c] += int(r[h.index(c)] or 0)
for k, name in (("P", "producer"), ("C", "consumer")):
    tot = sum(ops[k].values())
    print(f"{name}: {tot} warp-instr;  top ops:",
          ", ".join(f"{o} {v/tot:.1%}" for o, v in ops[k].most_common(10)))
    ts = sum(st[k].values()) or 1
    print(f"  stalls ({ts} samples):", ", ".join(f"{c[6:]} {v/ts:.1%}" for c, v in st[k].most_common(8)))
