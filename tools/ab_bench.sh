#!/bin/bash
# A/B of library variants on the driver-shaped bench (no e2e / cpu legs).
# usage (under gpurun): tools/ab_bench.sh TAG tree|variants/NAME.so ...  (REPS=2)
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for rep in $(seq ${REPS:-2}); do
  for lib in "$@"; do
    if [ "$lib" = tree ]; then L=""; else L="SFM_B200_LIB=$PWD/paper_2510_15271_b200/$lib"; fi
    env $L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/b.out 2>&1
    python - "$lib" $OUT/b.out <<'PY'
import json, sys
ln = [l for l in open(sys.argv[2]) if l.startswith('{')]
if not ln: print(sys.argv[1], "FAILED", open(sys.argv[2]).read()[-400:]); sys.exit()
d = json.loads(ln[-1]); k = d["kernels"]
print(f"{sys.argv[1]:24s} {d['value']:8.2f} it/s  " + " ".join(f"{n}={k[n]['ms']:.2f}" for n in list(k)[:8]))
PY
  done
done
