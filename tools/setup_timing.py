"""Wall-clock split of sfm_ba_solve's setup at config 3 (SFM_TIMING=1 marks on
stderr) over a few calls from pinned host arrays, plus the whole-call time."""
import os, sys, time
os.environ["SFM_TIMING"] = "1"
sys.path.insert(0, ".")
import numpy as np
import torch, dataclasses
from paper_2510_15271_b200.mapping import solve_arrays
from paper_2510_15271_b200.scenes import config_scene, scene_arrays
from paper_2510_15271_b200.solver import RobustLoss, SolverOptions
a = scene_arrays(config_scene(3, seed=0))
pin = {f.name: torch.from_numpy(getattr(a, f.name)).pin_memory().numpy() for f in dataclasses.fields(a)
       if isinstance(getattr(a, f.name), np.ndarray)}
a = dataclasses.replace(a, **pin)
for i in range(3):
    t0 = time.perf_counter()
    _, _, _, rep, raw = solve_arrays(a, RobustLoss("huber", 2.0), SolverOptions(max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 0))
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.2f} ms, device {raw.device_ms:.2f} ms, its {rep.iterations}", file=sys.stderr, flush=True)
