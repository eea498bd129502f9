"""Opcode histogram and hottest instructions of one kernel's ncu source page
(ncu -i REP --page source --csv -k regex:NAME). Diagnostic tool."""
import csv
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iw, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
seen, lst = set(), []
for r in rows[2:]:
    if len(r) <= iw or not r[iw].strip().isdigit() or r[ia] in seen:
        continue
    seen.add(r[ia])
    lst.append(r)
op, st, n, ns = Counter(), Counter(), 0, 0
for r in lst:
    t = r[isrc].split()
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    op[o] += int(r[ie] or 0)
    st[o] += int(r[iw] or 0)
    n += int(r[ie] or 0)
    ns += int(r[iw] or 0)
print("instructions", n, "stall samples", ns)
for o, v in op.most_common(22):
    print(f"{o:10s} {v:10d} {100*v/n:5.1f}%  stalls {100*st[o]/max(ns,1):5.1f}%")
print("hottest by stall samples:")
for r in sorted(lst, key=lambda r: -int(r[iw] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]:
    print(f"{lst.index(r):5d} {r[iw]:>6} {r[ie]:>9}  {r[isrc][:90]}")
