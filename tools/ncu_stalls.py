"""Stall-reason totals of one kernel from an ncu source page CSV (SASS view).
usage: ncu_stalls.py SRC.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
def f(x):
    try: return float(x)
    except: return 0.0
tot = {hdr[c][6:]: sum(f(r[c]) for r in data if len(r) > c) for c in cols}
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
    print(f"{k:28s} {100 * v / s:5.1f}%")
