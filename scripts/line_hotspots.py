"""Per-source-line stall samples from `ncu --page source --print-source cuda,sass --csv`."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for i, r in enumerate(rows):
    if r and r[0] == "Line No":
        hdr, start = r, i + 1
        break
ix_s = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
per_line = defaultdict(lambda: [0, "", defaultdict(int)])
cur = None
fname = ""
for r in rows[start:]:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) <= ix_s:
        continue
    if r[0].strip():
        if not r[0].strip().isdigit():
            cur = None
            continue
        cur = (fname, int(r[0]))
        per_line[cur][1] = r[1][:100]
    if cur is None:
        continue
    try:
        v = int(r[ix_s] or 0)
    except ValueError:
        continue
    per_line[cur][0] += v
    for k in stall_cols:
        try:
            per_line[cur][2][hdr[k][6:]] += int(r[k] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in per_line.values()) or 1
for ln, (v, src, st) in sorted(per_line.items(), key=lambda x: -x[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    top = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"{100*v/tot:5.1f}%  {ln[0][:18]}:{ln[1]:<5d} {src.strip()[:64]:64s} {', '.join(f'{k}={c}' for k, c in top)}")
