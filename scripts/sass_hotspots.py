"""Summarise an `ncu --page source --print-source sass --csv` dump: stall
reasons in total, instruction-class mix, and the top stalled instructions."""
import csv
import re
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for i, r in enumerate(rows):
    if len(r) > 5 and r[0] == "Address":
        hdr, start = r, i + 1
        break
ix = {h: k for k, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
mix = Counter()
top = []
for r in rows[start:]:
    if len(r) < len(hdr) or r[0] == "Address" or not r[0].startswith("0x"):
        continue
    src = r[ix["Source"]].strip()
    op = re.split(r"[ .]", src.lstrip("@!P0123456789 ").strip())[0] if src else "?"
    try:
        ex = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        ex = 0
    mix[op] += ex
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top.append((s, src))
    for c in stall_cols:
        try:
            tot[c] += int(r[ix[c]] or 0)
        except ValueError:
            pass
allsamp = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{k[6:]}={100*v/allsamp:.1f}%" for k, v in tot.most_common(8)))
te = sum(mix.values()) or 1
print("inst mix:", ", ".join(f"{k}={100*v/te:.1f}%" for k, v in mix.most_common(14)), f"(total {te})")
top.sort(reverse=True)
for s, src in top[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{s:7d}  {src}")
