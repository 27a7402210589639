"""Summarise a HIVC_DEBUG=timeline=<path> dump (decode.cu): per-lane I-solve windows, P-frame
busy time and the I-solve concurrency histogram of one decode call.

Usage: python tools/timeline.py tl.csv [block index, default -2]
"""
import collections
import sys


def main():
    blocks = [b for b in open(sys.argv[1]).read().split("-\n") if b.strip()]
    b = blocks[int(sys.argv[2]) if len(sys.argv) > 2 else -2]
    lanes = collections.defaultdict(list)
    for row in b.strip().split("\n"):
        l, k, s, g, f, t0, t1 = row.split(",")
        lanes[int(l)].append((float(t0), float(t1), k, int(s), int(g), int(f)))
    end = max(t1 for v in lanes.values() for _, t1, *_ in v)
    print(f"span {end:.0f} us, {len(blocks)} calls in file")
    for l in sorted(lanes):
        v = sorted(lanes[l])
        ints = [(t0, t1, s, g) for t0, t1, k, s, g, f in v if k == "I"]
        ps = [(t0, t1) for t0, t1, k, *_ in v if k == "P"]
        line = " ".join(f"I(s{s}g{g}) {t0:.0f}-{t1:.0f}" for t0, t1, s, g in ints)
        if ps:
            line += f" | P busy {sum(b - a for a, b in ps):.0f} first {min(a for a, _ in ps):.0f} last {max(b for _, b in ps):.0f}"
        print(l, line)
    ev = []
    for v in lanes.values():
        for t0, t1, k, *_ in v:
            if k == "I":
                ev += [(t0, 1), (t1, -1)]
    ev.sort()
    c, last, hist = 0, 0.0, collections.Counter()
    for t, d in ev:
        hist[c] += t - last
        c += d
        last = t
    print("I-solve concurrency (us):", {k: round(v) for k, v in sorted(hist.items())})


if __name__ == "__main__":
    main()
