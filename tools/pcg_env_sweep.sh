#!/bin/bash
# PCG variants via env knobs on config 3 (6 LM iterations each).
# usage: pcg_env_sweep.sh TAG "ENV1 ENV2 ..." "rtol:cluster ..."  (ENV like SFM_PCG_LOCAL=12,SFM_PCG_CTA=1024)
OUT=gpurun_out/$1; mkdir -p $OUT
for envs in $2; do
  for v in $3; do
    echo "env=$envs" >> $OUT/env_sweep.log
    env $(echo $envs | tr "," " ") timeout 300 python tools/pcg_sweep.py 3 ${ITERS:-6} $v >> $OUT/env_sweep.log 2>&1
  done
done
