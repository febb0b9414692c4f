"""Per source line: warp-instructions executed and stall samples, from
`ncu -i rep --page source --csv --print-source cuda,sass` (works without the
source files: line numbers come from -lineinfo).

    python tools/line_hot.py x.csv [top] [min_exec]
"""
import collections
import csv
import os
import sys

def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
rows = list(csv.reader(open(sys.argv[1])))
fname = None
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
hdr = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        continue
    d = dict(zip(hdr[2:], r[2:]))
    a = agg[cur]
    a[0] += num(d.get("Instructions Executed"))
    a[1] += num(d.get("Warp Stall Sampling (All Samples)"))
    a[2] += 1
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(f"warp-instructions {tot_i:.0f} samples {tot_s:.0f}")
srcs = {}
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2009_07174_b200/csrc/engine", f)
    if f not in srcs:
        srcs[f] = open(p).read().splitlines() if os.path.exists(p) else []
    line = srcs[f][ln - 1].strip()[:80] if ln - 1 < len(srcs[f]) else "?"
    print(f"{f:18s}:{ln:5d} ex {v[0]:11.0f} ({v[0] / tot_i * 100:4.1f}%) smp {v[1] / tot_s * 100:4.1f}%  sass {v[2]:4d}  {line}")
