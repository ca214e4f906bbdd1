"""Summarise an ncu --page source --csv --print-source sass dump: top
instructions by stall samples with their dominant stall reasons."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for r in data:
    for h in reasons:
        v = r[col[h]]
        if v.isdigit():
            tot[h] += int(v)
S = sum(tot.values())
print("total samples", S)
for h, v in tot.most_common(10):
    print(f"  {h:28s} {v:9d} {100*v/S:5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
key = col["Warp Stall Sampling (All Samples)"]
top = sorted(data, key=lambda r: -int(r[key]) if r[key].isdigit() else 0)[:n]
for r in top:
    rs = sorted(((int(r[col[h]]) if r[col[h]].isdigit() else 0, h[6:]) for h in reasons),
                reverse=True)[:2]
    print(f"{r[key]:>8} ex={r[col['Instructions Executed']]:>10} {r[col['Source']][:60]:60s} "
          + " ".join(f"{h}={v}" for v, h in rs))
