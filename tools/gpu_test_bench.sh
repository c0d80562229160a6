#!/bin/bash
# GPU parity tests + smoke + driver-shaped bench with the LM trace.
TAG=${1:-tb}; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
SFM_TRACE=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > $OUT/bench.out 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.out
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; grep -o '"value": [0-9.]*' $OUT/bench.out | head -1; grep -o '"kernels".*' $OUT/bench.out | cut -c1-900
