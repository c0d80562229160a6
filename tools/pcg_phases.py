"""Summarise per-CTA PCG phase cycles (library built with -DSFM_PCG_PHASES
-DSFM_PCG_PHASES_ALL) from the last solve in a log: mean / max over CTAs and
the correlation of each phase with the CTA's rows and blocks."""
import re
import sys

import numpy as np

rows = [l for l in open(sys.argv[1]) if l.startswith("PCGCTA")]
G = max(int(l.split()[1]) for l in rows) + 1
last = rows[-G:]
recs = []
for l in last:
    d = dict(re.findall(r"(\w+)=(\d+)", l))
    recs.append({k: int(v) for k, v in d.items()})
keys = ["spmv", "r1loop", "r1rpart", "r1bsum", "sync1", "gather", "coarse", "row2", "sync2", "zc"]
a = {k: np.array([r[k] for r in recs], float) for k in keys + ["rows", "blk"]}
print(f"G={G} rows mean {a['rows'].mean():.1f} max {a['rows'].max():.0f}  blocks mean {a['blk'].mean():.0f} "
      f"max {a['blk'].max():.0f}")
for k in keys:
    v = a[k]
    print(f"{k:8s} mean {v.mean():8.0f} max {v.max():8.0f} min {v.min():8.0f}  corr(rows) "
          f"{np.corrcoef(v, a['rows'])[0, 1]:+.2f} corr(blk) {np.corrcoef(v, a['blk'])[0, 1]:+.2f}")
work = a["spmv"] + a["r1loop"] + a["r1rpart"] + a["r1bsum"] + a["gather"] + a["coarse"] + a["row2"] + a["zc"]
print(f"non-barrier work per CTA: mean {work.mean():.0f} max {work.max():.0f}")
