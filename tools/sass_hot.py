"""Rank SASS instructions of an ncu source-page CSV by warp-stall samples.

    ncu -i rep --page source --csv --print-source sass [--launch-skip k --launch-count 1] > x.csv
    python tools/sass_hot.py x.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
col = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[col] or 0) for d in data)
ex = sum(float(d["Instructions Executed"] or 0) for d in data)
print(f"instructions {len(data)} samples {tot:.0f} warp-instructions executed {ex:.0f}")
idx = sorted(range(len(data)), key=lambda i: -float(data[i][col] or 0))[:top]
for i in sorted(idx):
    d = data[i]
    print(f"{i:6d} {float(d[col]) / tot * 100:5.1f}% ex {d['Instructions Executed']:>10} {d['Source'].strip()[:90]}")
