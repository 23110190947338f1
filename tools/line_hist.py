"""Per-CUDA-source-line instruction attribution from an ncu
`--page source --csv --print-source cuda,sass` export.
usage: line_hist.py mixed.csv [per_iter_divisor] [top]"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
cur = None; agg = defaultdict(int); text = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if len(r) > 3 and r[0] == "Line No":
        ie = r.index("Instructions Executed"); continue
    if cur and len(r) > 10:
        try: ln = int(r[0])
        except ValueError: continue
        try: v = int(r[ie])
        except ValueError: v = 0
        agg[(cur, ln)] += v; text[(cur, ln)] = r[1][:110]
tot = sum(agg.values()); print("total", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / tot * 100:5.1f}% {v / div:7.1f} {k[0]}:{k[1]} {text[k].strip()}")
