"""Host-side split of the e2e call on config 3: setup (H2D + structure
build + initial cost), LM iterations, download.  SFM_TIMING=1 adds the
per-phase split of sfm_ba_setup on stderr."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2510_15271_b200.scenes import config_scene, scene_arrays
from paper_2510_15271_b200.mapping import DeviceBA, solve_arrays
from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions
a = scene_arrays(config_scene(int(sys.argv[1]) if len(sys.argv) > 1 else 3, seed=0))
import dataclasses, torch
a = dataclasses.replace(a, **{f.name: torch.from_numpy(getattr(a, f.name)).pin_memory().numpy()
                              for f in dataclasses.fields(a) if isinstance(getattr(a, f.name), np.ndarray)})
loss = RobustLoss("huber", 2.0)
dopt = DeviceOptions(linear_solver="pcg", pcg_rtol=1e-8, pcg_max_iters=500)
for rep in range(2):
    t0 = time.perf_counter(); ba = DeviceBA(a, loss, SolverOptions(max_iters=10), dopt)
    t1 = time.perf_counter(); r = ba.iterate(10)
    t2 = time.perf_counter(); ba.download()
    t3 = time.perf_counter()
    print(f"setup {1e3*(t1-t0):.1f} ms  iterate {1e3*(t2-t1):.1f} ms (device {r.device_ms:.1f})  download {1e3*(t3-t2):.1f} ms", flush=True)
    del ba
t0 = time.perf_counter(); out = solve_arrays(a, loss, SolverOptions(max_iters=10), dopt); t1 = time.perf_counter()
print(f"solve_arrays total {1e3*(t1-t0):.1f} ms", flush=True)
