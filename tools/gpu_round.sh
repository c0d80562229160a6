#!/bin/bash
# One GPU call: gpu parity tests, smoke, bench (N=1), ncu launch list + full capture of the top kernel.
# usage (under gpurun): bash tools/gpu_round.sh [tag] [full-kernel-regex]
TAG=${1:-r1}
KRE=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> $OUT/nproc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_bench.log 2>&1
if [ -n "$KRE" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 3 -c 2 \
     -o $OUT/prof python tools/ncu_target.py 3 2 > $OUT/ncu_full.log 2>&1
fi
tail -3 $OUT/*.log
