#!/bin/bash
# k_ransac (one track per warp) vs k_ransac_packed (up to three short tracks
# per warp): ncu kernel times inside configs[1] / configs[3] iterative_map.
# usage (under gpurun): tools/ransac_pack_ab.sh TAG variants/nopack.so
OUT=gpurun_out/$1; mkdir -p $OUT
for lib in tree $2; do
  if [ "$lib" = tree ]; then L=""; else L="SFM_B200_LIB=$PWD/paper_2510_15271_b200/$lib"; fi
  for cfg in 2 4; do
    env $L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_ransac" --csv \
      --log-file $OUT/$(basename $lib .so)_cfg$cfg.csv python tools/imap_run.py $cfg 1 > /dev/null 2>&1
    python - $OUT/$(basename $lib .so)_cfg$cfg.csv "$lib cfg$cfg" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
vals = [float(r[h.index("Metric Value")].replace(",", "")) for r in rows[1:]]
print(sys.argv[2], "launches", len(vals), "first ms %.3f" % (vals[0] / 1e6), "total ms %.3f" % (sum(vals) / 1e6))
PY
  done
done
