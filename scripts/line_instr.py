"""Per-source-line executed (warp) instructions from an ncu cuda,sass source CSV."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
per = defaultdict(lambda: [0, ""])
fname, cur, hdr, ie = "", None, None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if not hdr or len(r) <= ie:
        continue
    if r[0].strip():
        if not r[0].strip().isdigit():
            cur = None
            continue
        cur = (fname, int(r[0]))
        per[cur][1] = r[1][:90]
    if cur is None:
        continue
    try:
        per[cur][0] += int(r[ie] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in per.values()) or 1
print("total warp instructions (double-counted listing /2):", tot // 2)
for k, v in sorted(per.items(), key=lambda x: -x[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{100*v[0]/tot:5.1f}% {k[0][:18]}:{k[1]:<5d} {v[1].strip()[:90]}")
