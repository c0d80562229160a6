#!/bin/bash
# A/B: the same config-3 LM sweep with each library variant (SFM_B200_LIB).
# usage: tools/ab_run.sh TAG lib1.so lib2.so ...   (in-tree lib = "tree")
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for rep in 1 2; do
  for lib in "$@"; do
    echo "env=lib:$lib" >> $OUT/env_sweep.log
    if [ "$lib" = tree ]; then L=""; else L="SFM_B200_LIB=$PWD/$lib"; fi
    env $L timeout 300 python tools/pcg_sweep.py 3 ${ITERS:-6} 1e-10:8 >> $OUT/env_sweep.log 2>&1
  done
done
