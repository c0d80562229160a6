#!/bin/bash
# A/B of runtime env knobs on the bench (whole solves; no e2e / cpu / extra legs).
# usage (under gpurun): tools/ab_env.sh TAG "ENV1=a ENV2=b" "ENV3=c" ...   ("-" = no env)
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for rep in $(seq ${REPS:-2}); do
  for e in "$@"; do
    if [ "$e" = "-" ]; then E=""; else E="$e"; fi
    env $E timeout 300 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --no-extra ${MAXIT:+--max-iters $MAXIT} > $OUT/b.out 2>&1
    python - "$e" $OUT/b.out <<'PY'
import json, sys
ln = [l for l in open(sys.argv[2]) if l.startswith('{')]
if not ln: print(sys.argv[1], "FAILED", open(sys.argv[2]).read()[-400:]); sys.exit()
d = json.loads(ln[-1]); k = d["kernels"]
top = sorted(k.items(), key=lambda kv: -kv[1]["avg_ms"] * kv[1]["launches"])[:7]
print(f"{sys.argv[1]:34s} {d['value']:8.2f} it/s its={d['iterations_per_solve']} tr={d['trials_per_solve']} pcg={d['pcg_iterations_per_solve']} "
      f"cost={d['cost']['final']!r} {d['cost']['termination']} | " +
      " ".join(f"{n}={v['avg_ms'] * v['launches']:.2f}" for n, v in top), flush=True)
PY
  done
done
