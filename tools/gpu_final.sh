#!/bin/bash
# Round-end evidence in one GPU call: gpu tests, smoke, the driver-shaped
# bench (with the sfmkit CPU baseline), the reference arm, the ncu launch
# list (DRAM bytes) and one --set full capture of the top kernels.
TAG=${1:-fin}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> $OUT/nproc.txt
if [ "${TESTS:-1}" = "1" ]; then
  timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench.out 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
if [ "${REF:-1}" = "1" ]; then
  timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref.out 2> $OUT/bench_ref.err; echo "ref rc=$?" >> $OUT/bench_ref.err
fi
if [ "${PROFILE:-1}" = "1" ]; then bash tools/gpu_profile.sh $TAG; fi
tail -3 $OUT/pytest_gpu.log 2>/dev/null; tail -2 $OUT/smoke.log; head -c 600 $OUT/bench.out; echo; head -c 400 $OUT/bench_ref.out 2>/dev/null
