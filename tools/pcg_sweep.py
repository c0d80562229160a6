"""PCG sweep on a config scene: LM progress vs PCG work for tolerance /
coarse-cluster variants.  usage: pcg_sweep.py CFG ITERS [rtol:cluster ...]"""
import sys, time, json
sys.path.insert(0, ".")
from paper_2510_15271_b200.scenes import config_scene, scene_arrays
from paper_2510_15271_b200.mapping import DeviceBA
from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
variants = [(float(v.split(":")[0]), int(v.split(":")[1])) for v in sys.argv[3:]] or \
    [(1e-12, 16), (1e-6, -1), (1e-6, 16), (1e-6, 8), (1e-6, 32)]
sc = config_scene(cfg, seed=0)
a = scene_arrays(sc)
for rtol, cl in variants:
    ba = DeviceBA(a, RobustLoss("huber", 2.0), SolverOptions(max_iters=100),
                  DeviceOptions(linear_solver="pcg", pcg_rtol=rtol, pcg_max_iters=20000,
                                coarse_cluster=cl))
    ba.ctx.set_profiling(True)
    ba.ctx.reset_profile()
    costs, tot_ms = [], 0.0
    for k in range(iters):
        r = ba.iterate(1)
        tot_ms += r.device_ms
        costs.append((r.final_cost, r.n_trials, r.pcg_iterations))
    prof = {k: round(v["ms"], 3) for k, v in ba.ctx.profile().items()}
    ba.ctx.set_profiling(False)
    print(json.dumps({"rtol": rtol, "cluster": cl, "ms": tot_ms, "costs": costs, "prof": prof}), flush=True)
