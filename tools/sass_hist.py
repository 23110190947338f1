"""Summarise an ncu `--page source --csv --print-source sass` export: total warp
instructions, the execution-count classes (hot loop vs rare paths) and a raw
metrics excerpt.  usage: sass_hist.py src.csv [raw.csv]"""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = [r for r in rows[2:] if len(r) == len(h)]
ie = h.index("Instructions Executed")
def n(x):
    try: return int(x)
    except ValueError: return 0
tot = sum(n(r[ie]) for r in data)
print("total warp inst", tot, "static", len(data))
c = Counter(n(r[ie]) for r in data)
for k, v in sorted(c.items(), key=lambda x: -x[0] * x[1])[:12]:
    print(k, v, k * v, round(k * v / tot, 3))
if len(sys.argv) > 2:
    raw = list(csv.reader(open(sys.argv[2])))
    hh, vv = raw[0], raw[2]
    for key in ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]:
        if key in hh: print(key, vv[hh.index(key)])
