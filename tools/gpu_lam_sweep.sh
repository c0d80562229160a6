#!/bin/bash
# Coarse-level policy sweep on the driver-shaped bench (trace on stderr).
TAG=${1:-ls}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for cfg in "1e-2 4" "1e-4 4" "1e-3 4" "1e-1 4" "1e-2 16" "1e-2 2" "1e-8 4"; do
  set -- $cfg
  SFM_TRACE=1 SFM_COARSE_LAMMAX=$1 SFM_COARSE_DRIFT=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
     > $OUT/b_$1_$2.out 2> $OUT/b_$1_$2.err
  echo "$1 $2 $(grep -o '"value": [0-9.]*' $OUT/b_$1_$2.out | head -1) $(grep -o '"pcg_iterations_timed": [0-9]*' $OUT/b_$1_$2.out)"
done
