"""Top SASS instructions by warp-stall samples from an ncu source page CSV
(ncu -i X.ncu-rep --page source --csv --kernel-name regex:K --print-source sass)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = rows[2:]
ci = hdr.index("Warp Stall Sampling (All Samples)")
si = hdr.index("Source"); ai = hdr.index("Address")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
def f(x):
    try: return float(x)
    except: return 0.0
tot = sum(f(r[ci]) for r in data)
print(f"total samples {tot:.0f}")
idx = sorted(range(len(data)), key=lambda i: -f(data[i][ci]))[:top]
for i in sorted(idx):
    r = data[i]
    st = sorted(((f(r[c]), hdr[c][6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{i:5d} {100*f(r[ci])/tot:5.1f}%  {r[si][:60]:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0))
