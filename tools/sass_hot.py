"""Hot SASS listing in address order from an ncu mixed (cuda,sass) source
export: every instruction executed >= min_frac of the max count, with its
per-iteration count and source line.  usage: sass_hot.py mixed.csv div [min_frac]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]); mf = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
hdr = None; src = None; cur = None; ins = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if len(r) > 3 and r[0] == "Line No": hdr = r; ie = r.index("Instructions Executed"); continue
    if not hdr or len(r) != len(hdr): continue
    if r[0]: src = f"{cur}:{r[0]}"; continue
    if r[2].startswith("0x"):
        try: n = int(r[ie])
        except ValueError: n = 0
        ins.append((int(r[2], 16), n, r[3].strip(), src))
ins.sort()
mx = max(n for _, n, _, _ in ins)
tot = 0
for a, n, t, s in ins:
    if n >= mf * mx:
        tot += n
        print(f"{a & 0xffff:05x} {n / div:6.2f} {t[:70]:70s} {s}")
print("hot total per iter", round(tot / div, 1))
