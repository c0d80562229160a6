"""iterative_map on a config scene (tracks = the generated observations,
initial poses = the perturbed ones): outcome, rounds and timing."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2510_15271_b200.scenes import config_scene, make_scene
from paper_2510_15271_b200.cameras import CameraModel
from paper_2510_15271_b200.mapping import MappingConfig, iterative_map_arrays, model_table
from paper_2510_15271_b200.solver import DeviceOptions

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sc = config_scene(cfg, seed=0)
models, n_models, fm = model_table([CameraModel(**sc.camera)] * sc.n_frames)
ptr = np.searchsorted(sc.obs_point, np.arange(sc.n_points + 1)).astype(np.int64)
F = sc.n_frames
edges = np.stack([np.arange(F - 1), np.arange(1, F)], 1).astype(np.int32)
priors = np.flatnonzero(sc.frame_fixed == 0).astype(np.int32)
dev = DeviceOptions()  # drop-in defaults, as bench.py
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    t0 = time.perf_counter()
    try:
        r = iterative_map_arrays(sc.cam_q, sc.cam_t, fm, sc.frame_fixed, models, n_models, ptr,
                                 sc.obs_frame, sc.obs_uv, edges, priors, MappingConfig(), device=dev)
        dt = time.perf_counter() - t0
        print(f"config {cfg}: {sc.n_frames} frames {sc.n_points} tracks {len(sc.obs_frame)} obs: "
              f"{dt:.2f} s, landmarks {len(r.lm_track)}, stats {r.round_stats}", flush=True)
    except Exception as e:
        print(f"config {cfg}: {type(e).__name__}: {e} after {time.perf_counter() - t0:.2f} s", flush=True)
