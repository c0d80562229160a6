"""Cost of the cross-launch barrier of the row-partitioned PCG, measured on
one device: the config-3 solve point-sharded over emulated ranks with one
PCG launch over all ranks' CTAs (pcg_partition 1, grid barrier) vs one
launch per rank meeting at the cross-launch barrier (pcg_partition 2).
Same arithmetic, so the time difference over the PCG iterations is the
barrier's extra cost.  usage: xbar_cost.py [ranks] [LM iterations]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2510_15271_b200.mapping import solve_sharded_emulated
from paper_2510_15271_b200.scenes import config_scene, scene_arrays
from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions
R = int(sys.argv[1]) if len(sys.argv) > 1 else 2
its = int(sys.argv[2]) if len(sys.argv) > 2 else 5
a = scene_arrays(config_scene(3, seed=0))
loss, sopt = RobustLoss("huber", 2.0), SolverOptions(max_iters=its)
res = {}
for mode in (1, 2, 1, 2):
    dopt = DeviceOptions(pcg_partition=mode)
    t0 = time.perf_counter()
    q, t, X, rep, raw = solve_sharded_emulated(a, loss, sopt, dopt, R)
    dt = time.perf_counter() - t0
    res.setdefault(mode, []).append((raw.device_ms, raw.pcg_iterations, rep.final_cost, dt))
    print(f"ranks {R} pcg_partition {mode}: device {raw.device_ms:.2f} ms, {raw.pcg_iterations} PCG it, "
          f"cost {rep.final_cost!r}, wall {dt:.2f} s", flush=True)
d1 = min(r[0] for r in res[1]); d2 = min(r[0] for r in res[2]); n = res[1][0][1]
print(f"cross-launch barrier: {(d2 - d1) * 1e3 / max(n, 1) / 2:.2f} us extra per barrier "
      f"({d2 - d1:.2f} ms over {n} PCG iterations, 2 barriers each)")
