"""Per-CUDA-source-line warp-stall samples from an ncu `--page source --csv
--print-source cuda,sass` export, with the dominant stall reasons per line.
usage: stall_hist.py mixed.csv [top]"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = None; agg = defaultdict(float); reasons = defaultdict(lambda: defaultdict(float)); text = {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r; ws = r.index("Warp Stall Sampling (All Samples)")
        st = [(i, h) for i, h in enumerate(r) if h.startswith("stall_")]
        continue
    if cur and hdr and len(r) == len(hdr):
        try: ln = int(r[0])
        except ValueError: continue
        try: v = float(r[ws])
        except ValueError: v = 0
        agg[(cur, ln)] += v; text[(cur, ln)] = r[1][:90]
        for i, h in st:
            try: reasons[(cur, ln)][h] += float(r[i])
            except ValueError: pass
tot = sum(agg.values()); print("total samples", tot)
tr = defaultdict(float)
for k in reasons:
    for h, v in reasons[k].items(): tr[h] += v
print("by reason:", ", ".join(f"{h[6:]} {v / tot * 100:.1f}%" for h, v in sorted(tr.items(), key=lambda x: -x[1])[:8]))
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    rs = sorted(reasons[k].items(), key=lambda x: -x[1])[:2]
    print(f"{v / tot * 100:5.1f}% {k[0]}:{k[1]} [{', '.join(f'{h[6:]} {x / max(v, 1) * 100:.0f}%' for h, x in rs)}] {text[k].strip()}")
