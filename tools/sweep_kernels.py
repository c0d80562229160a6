import json, sys
hdr = ""
keys = sys.argv[2].split(",") if len(sys.argv) > 2 else ["pcg", "schur_offdiag", "schur_diag", "point_lin", "point_trial", "cam_lin"]
for ln in open(sys.argv[1]):
    if ln.startswith('env'): hdr = ln.strip(); continue
    if not ln.startswith('{'): print(ln[:300].rstrip()); continue
    d = json.loads(ln)
    print(f"{hdr:40s} ms {d['ms']:.2f} " + " ".join(f"{k}={d['prof'].get(k, 0):.3f}" for k in keys))
