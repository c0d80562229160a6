#!/bin/bash
# One GPU call: L2 stream peak, gpu tests (optional), smoke, bench (driver flags), e2e breakdown.
# usage (under gpurun): bash tools/gpu_bench2.sh TAG [tests:0|1] [extra bench flags]
TAG=${1:-b2}; TESTS=${2:-1}; shift; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2stream tools/micro/l2stream.cu > $OUT/l2stream.log 2>&1 && /tmp/l2stream >> $OUT/l2stream.log 2>&1
nproc > $OUT/nproc.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> $OUT/nproc.txt
if [ "$TESTS" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
SFM_TRACE=1 timeout 1200 python bench.py --steps 20 --warmup 5 "$@" > $OUT/bench.out 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.out
tail -3 $OUT/pytest_gpu.log 2>/dev/null; tail -2 $OUT/smoke.log; cat $OUT/l2stream.log; head -c 1500 $OUT/bench.out; tail -3 $OUT/bench.err
