#!/bin/bash
# GPU call: the config-scale parity tests (or PYTEST_K) + the profiling pass (tools/gpu_profile.sh).
TAG=${1:-pp}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-config3_lm or config2_iterative_map_matches}" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -30 $OUT/pytest_gpu.log
[ "${PROFILE:-1}" = "1" ] && bash tools/gpu_profile.sh $TAG
