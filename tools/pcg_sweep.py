"""PCG tolerance sweep on the config-3 scene: LM progress vs PCG work."""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np
from paper_2510_15271_b200.scenes import config_scene, scene_arrays
from paper_2510_15271_b200.mapping import DeviceBA
from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
sc = config_scene(cfg, seed=0)
a = scene_arrays(sc)
for rtol, mx in [(1e-12, 20000), (1e-8, 5000), (1e-6, 5000), (1e-4, 5000), (1e-2, 5000)]:
    ba = DeviceBA(a, RobustLoss("huber", 2.0), SolverOptions(max_iters=100),
                  DeviceOptions(linear_solver="pcg", pcg_rtol=rtol, pcg_max_iters=mx))
    costs = []
    t0 = time.time()
    tot_ms = 0.0
    for k in range(iters):
        r = ba.iterate(1)
        tot_ms += r.device_ms
        costs.append((r.final_cost, r.n_trials, r.pcg_iterations))
    print(json.dumps({"rtol": rtol, "ms": tot_ms, "costs": costs}), flush=True)
