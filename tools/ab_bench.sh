#!/bin/bash
# A/B of library variants on the bench (whole solves; no e2e / cpu / extra legs).
# usage (under gpurun): tools/ab_bench.sh TAG tree|variants/NAME.so ...  (REPS=2)
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for rep in $(seq ${REPS:-2}); do
  for lib in "$@"; do
    if [ "$lib" = tree ]; then L=""; else L="SFM_B200_LIB=$PWD/paper_2510_15271_b200/$lib"; fi
    env $L timeout 300 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --no-extra ${MAXIT:+--max-iters $MAXIT} > $OUT/b.out 2>&1
    python - "$lib" $OUT/b.out <<'PY'
import json, sys
ln = [l for l in open(sys.argv[2]) if l.startswith('{')]
if not ln: print(sys.argv[1], "FAILED", open(sys.argv[2]).read()[-600:]); sys.exit()
d = json.loads(ln[-1]); k = d["kernels"]
top = sorted(k.items(), key=lambda kv: -kv[1]["avg_ms"] * kv[1]["launches"])[:8]
print(f"{sys.argv[1]:26s} {d['value']:8.2f} it/s its={d['iterations_per_solve']} tr={d['trials_per_solve']} pcg={d['pcg_iterations_per_solve']} "
      f"cost={d['cost']['final']!r} {d['cost']['termination']} | " +
      " ".join(f"{n}={v['avg_ms']:.4f}" for n, v in top), flush=True)
PY
  done
done
