#!/bin/bash
# One ncu --set full capture of the LM kernels at config 3 (LM iteration 4-5),
# source-level stall sampling on.  usage (under gpurun): gpu_ncu_full.sh TAG [kernel regex] [skip] [count]
TAG=${1:-nf}; OUT=gpurun_out/$TAG; mkdir -p $OUT
KRE=${2:-"k_pcg3|k_offdiag_blocks|k_cam_blocks|k_point_lin|k_point_cost|k_point_prep"}
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$KRE" -s ${3:-24} -c ${4:-7} \
   -o $OUT/full python tools/ncu_target.py 3 5 > $OUT/full.log 2>&1
echo "ncu rc=$?"; tail -3 $OUT/full.log
