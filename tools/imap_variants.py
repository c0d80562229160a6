"""iterative_map on config-4-sized scenes with generator variants (shape,
depth range, seed): which raise NonPositiveDepth out of a BA trial."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2510_15271_b200.scenes import CONFIGS, make_scene
from paper_2510_15271_b200.cameras import CameraModel
from paper_2510_15271_b200.mapping import MappingConfig, iterative_map_arrays, model_table

for shape, depth, seed in [("curve", (1.0, 40.0), 1), ("curve", (2.0, 40.0), 0), ("curve", (3.0, 40.0), 0),
                           ("line", (3.0, 40.0), 0)]:
    args = dict(CONFIGS[4]); args.update(shape=shape, depth=depth)
    sc = make_scene(seed=seed, **args)
    models, n_models, fm = model_table([CameraModel(**sc.camera)] * sc.n_frames)
    ptr = np.searchsorted(sc.obs_point, np.arange(sc.n_points + 1)).astype(np.int64)
    F = sc.n_frames
    edges = np.stack([np.arange(F - 1), np.arange(1, F)], 1).astype(np.int32)
    priors = np.flatnonzero(sc.frame_fixed == 0).astype(np.int32)
    t0 = time.perf_counter()
    try:
        r = iterative_map_arrays(sc.cam_q, sc.cam_t, fm, sc.frame_fixed, models, n_models, ptr,
                                 sc.obs_frame, sc.obs_uv, edges, priors, MappingConfig())
        print(f"{shape} {depth} seed {seed}: {sc.n_points} tracks {sc.n_obs} obs: {time.perf_counter() - t0:.2f} s, "
              f"landmarks {len(r.lm_track)}, stats {r.round_stats}", flush=True)
    except Exception as e:
        print(f"{shape} {depth} seed {seed}: {type(e).__name__}: {e} after {time.perf_counter() - t0:.2f} s", flush=True)
