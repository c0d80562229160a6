#!/bin/bash
# Driver-shaped bench (--steps 20 --warmup 5) with the per-trial LM trace on stderr.
# usage (under gpurun): bash tools/gpu_bench_trace.sh TAG [extra bench args]
TAG=${1:-bt}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
SFM_TRACE=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > $OUT/bench.out 2> $OUT/bench.err
echo "bench rc=$?" >> $OUT/bench.out
grep -c "sfm trial" $OUT/bench.err; tail -c 1500 $OUT/bench.out
