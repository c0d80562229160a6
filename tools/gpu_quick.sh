#!/bin/bash
# Quick GPU check: parity tests + bench (no cpu baseline) + optional pcg sweep.
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
if [ -n "$2" ]; then timeout 900 python tools/pcg_sweep.py 3 4 $2 > $OUT/sweep.log 2>&1; fi
tail -3 $OUT/pytest_gpu.log; grep -o '"value": [0-9.]*' $OUT/bench.log | head -1; grep -o '"kernels".*' $OUT/bench.log | cut -c1-900
