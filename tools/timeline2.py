"""Print one decode call of a HIVC_DEBUG=timeline=<path> dump per item: host I-parse (H),
batched I-solve (I), finalize (F), host P-phase (Q), P-frame kernels (P).

Usage: python tools/timeline2.py tl.csv [call index, default -2]
"""
import collections
import sys

blocks = [b for b in open(sys.argv[1]).read().split("-\n") if b.strip()]
b = blocks[int(sys.argv[2]) if len(sys.argv) > 2 else -2]
by = collections.defaultdict(list)
for row in b.strip().split("\n"):
    l, k, s, g, f, t0, t1 = row.split(",")
    by[int(l)].append((k, int(s), int(g), float(t0), float(t1)))
for l in sorted(by):
    ev = by[l]
    s, g = ev[0][1], ev[0][2]
    parts = []
    for k in "HIFQD":
        for kk, _, _, a, bb in ev:
            if kk == k:
                parts.append(f"{k} {a / 1e3:6.2f}-{bb / 1e3:6.2f}")
    ps = [(a, bb) for kk, _, _, a, bb in ev if kk == "P"]
    if ps:
        parts.append(f"P {min(a for a, _ in ps) / 1e3:6.2f}-{max(bb for _, bb in ps) / 1e3:6.2f} busy {sum(bb - a for a, bb in ps) / 1e3:5.2f}")
    print(f"item {l:2d} s{s}g{g}: " + " | ".join(parts))
