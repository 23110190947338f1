"""Format an ncu `--metrics gpu__time_duration.sum --csv` launch list:
one line per launch (kernel, duration) plus per-kernel totals.
usage: launch_list.py launches.csv"""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = defaultdict(float); cnt = defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum": continue
    v = float(r[vi].replace(",", "")); u = r[ui]
    ms = v / 1e6 if u == "ns" else v / 1e3 if u in ("us", "usecond") else v if u in ("ms", "msecond") else v / 1e6
    name = r[ki].split("(")[0][:70]
    print(f"{name:72s} {ms:9.3f} ms")
    tot[name] += ms; cnt[name] += 1
print("--- totals")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:72s} {cnt[k]:4d} launches {v:9.3f} ms")
