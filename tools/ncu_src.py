"""Summarise an ncu --page source --csv dump: top SASS lines by stall samples + stall totals."""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
hi = [i for i, row in enumerate(r) if "Source" in row and "Address" in row][0]
h = r[hi]
rows = [dict(zip(h, x)) for x in r[hi + 1:] if len(x) == len(h)]
S = "Warp Stall Sampling (All Samples)"
tot = sum(int(x[S] or 0) for x in rows)
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(int(x[c] or 0) for x in rows) for c in stalls}
print("total samples", tot)
for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]:
    print(f"  {c:28s} {v:8d} {100 * v / max(tot, 1):5.1f}%")
top = sorted(rows, key=lambda x: -int(x[S] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for x in top:
    print(f"{int(x[S]):7d} {x['Address'][-5:]} {x['Source'].strip()[:90]}")
