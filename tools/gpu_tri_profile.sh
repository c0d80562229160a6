#!/bin/bash
# ncu counters of the triangulation / gating kernels inside configs[1] and
# configs[3] iterative_map (fp64 instruction counts -> achieved FLOP/s vs the
# measured DFMA peak; DRAM bytes -> GB/s vs HBM).  usage: gpu_tri_profile.sh TAG
OUT=gpurun_out/$1; mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for cfg in 2 4; do
  timeout 900 ncu --metrics $M --clock-control none -k "regex:k_ransac|k_gate|k_rays" --csv --log-file $OUT/tri_cfg$cfg.csv \
     python tools/imap_run.py $cfg 1 > $OUT/tri_cfg$cfg.log 2>&1
done
for f in $OUT/tri_cfg*.log; do tail -n 2 $f; done
