"""Small driver for ncu captures: LM iterations on a config scene with the
bench's solver options (bench.py), one iterate() call per LM iteration so
the per-iteration PCG counts can be matched to captured launches.
usage: ncu_target.py [CFG] [ITERS]"""
import sys
sys.path.insert(0, ".")
from paper_2510_15271_b200.scenes import config_scene, scene_arrays
from paper_2510_15271_b200.mapping import DeviceBA
from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
a = scene_arrays(config_scene(cfg, seed=0))
ba = DeviceBA(a, RobustLoss("huber", 2.0), SolverOptions(), DeviceOptions())  # bench.py's (drop-in defaults)
prev = 0
for i in range(iters):
    r = ba.iterate(1)
    print(f"LM iteration {r.iterations}: trials {r.n_trials} pcg iterations {r.pcg_iterations - prev} "
          f"device {r.device_ms:.3f} ms", flush=True)
    prev = r.pcg_iterations
