# grouped vs staged RANSAC: identical outputs on config-2/4 tracks, and timing
import sys, time, os
sys.path.insert(0, ".")
import numpy as np
from paper_2510_15271_b200.scenes import config_scene
from paper_2510_15271_b200 import _native as nat
import ctypes
sys.path.insert(0, "tests")
from test_gpu_configs import tracks_from_scene
for cfg in (2, 4):
    sc = config_scene(cfg, seed=0)
    s, keep = tracks_from_scene(sc)
    ctx = nat.default_context()
    T, N = sc.n_points, len(sc.obs_frame)
    X = np.empty((T, 3)); mask = np.empty(N, np.uint8); st = np.empty(T, np.int8)
    for rep in range(3):
        t0 = time.perf_counter()
        ctx.check(ctx.lib.sfm_ransac_triangulate(ctx.handle, ctypes.byref(s), 4.0, float(np.radians(0.5)), 0, nat.ptr(X), nat.ptr(mask), nat.ptr(st)))
        dt = time.perf_counter() - t0
    np.savez(f"gpurun_out/rs_{os.environ.get('TAG','x')}_{cfg}.npz", X=X, mask=mask, st=st)
    print(cfg, f"{dt*1e3:.1f} ms", np.bincount(st), flush=True)
