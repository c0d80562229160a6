#!/bin/bash
# configs[1] / configs[3] iterative_map wall time (second run) per library variant.
# usage (under gpurun): tools/imap_ab.sh tree variants/NAME.so ...
for lib in "$@"; do
  if [ "$lib" = tree ]; then L=""; else L="SFM_B200_LIB=$PWD/paper_2510_15271_b200/$lib"; fi
  for cfg in 2 4; do echo "$lib cfg$cfg: $(env $L timeout 900 python tools/imap_run.py $cfg 2 2>&1 | tail -n 1 | cut -c1-100)"; done
done
