#!/bin/bash
# Profiling call: launch list of a short bench run + one full ncu capture of
# the top kernels at LM iteration 4 (config 3).  usage: gpu_profile.sh TAG
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extra > $OUT/launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
   -k "regex:k_pcg3|k_offdiag_blocks|k_cam_fma|k_cam_blocks|k_point_lin|k_point_cost|k_gj_inverse|k_point_prep" \
   -s 24 -c 9 -o $OUT/full python tools/ncu_target.py 3 5 > $OUT/full.log 2>&1
tail -3 $OUT/full.log
