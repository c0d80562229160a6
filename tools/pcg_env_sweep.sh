#!/bin/bash
# PCG variants via env knobs on config 3 (4 LM iterations each).
OUT=gpurun_out/$1; mkdir -p $OUT
for cta in 512 1024; do
  for rf in 1 4; do
    for cl in 16 8; do
      echo "cta=$cta refresh=$rf" >> $OUT/env_sweep.log
      SFM_PCG_CTA=$cta SFM_COARSE_REFRESH=$rf timeout 300 python tools/pcg_sweep.py 3 6 1e-10:$cl >> $OUT/env_sweep.log 2>&1
    done
  done
done
