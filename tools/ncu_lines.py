"""Aggregate warp-stall samples per CUDA source line from
`ncu -i rep --page source --csv --print-source cuda,sass` output."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
agg = collections.Counter()
src = {}
fname = None
hdr = None
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:  # a CUDA source line row
        line = (fname, r[0])
        src[line] = r[1].strip()
    try:
        s = int(r[4] or 0)
    except ValueError:
        continue
    if line is not None and not r[0]:
        agg[line] += s
tot = sum(agg.values())
print("total samples", tot)
for (f, ln), s in agg.most_common(top):
    print(f"{s:7d} {100 * s / max(tot, 1):5.1f}% {f}:{ln:>5}  {src.get((f, ln), '')[:90]}")
