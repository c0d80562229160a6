"""compute-sanitizer memcheck / racecheck / synccheck over the device paths
(the persistent cooperative kernels -- k_pcg3 and
k_gj_inverse with their grid barriers -- the DMMA Schur kernels, the
matrix-free Schur PCG, RANSAC and gating) on small problems: the
byte-identical determinism contract (test_acceptance.py:603-637) rests on
the absence of races."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKLOAD = r"""
import sys
sys.path.insert(0, %r)
import numpy as np
from paper_2510_15271_b200.cameras import CameraModel
from paper_2510_15271_b200.mapping import MappingConfig, iterative_map_arrays, model_table, solve_arrays
from paper_2510_15271_b200.scenes import config_scene, make_scene, scene_arrays
from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions
huber = RobustLoss("huber", 2.0)
# configs[0]: the dense reduced solve
_, _, _, rep, _ = solve_arrays(scene_arrays(config_scene(1, seed=0)), huber, SolverOptions(max_iters=4))
print("config1", rep.termination, rep.final_cost)
# two-level PCG (coarse Gauss-Jordan + persistent PCG), then the matrix-free
# Schur PCG of the high-damping trials (lambda0 = 1e3)
sc = make_scene(64, 4000, 20000, shape="line", seed=2)
a = scene_arrays(sc)
dev = DeviceOptions(linear_solver="pcg", coarse_cluster=4)
_, _, _, rep, raw = solve_arrays(a, huber, SolverOptions(max_iters=3), dev)
print("pcg", rep.termination, rep.final_cost, raw.pcg_iterations)
_, _, _, rep, raw = solve_arrays(a, huber, SolverOptions(max_iters=3, initial_lambda=1e3), dev)
print("pcg high damping", rep.termination, rep.final_cost, raw.pcg_iterations)
# point-sharded over 3 emulated ranks: reduce-scatter of S by block rows and
# the row-partitioned PCG in one launch over every rank's CTAs
from paper_2510_15271_b200.mapping import solve_sharded_emulated
_, _, _, rep, raw = solve_sharded_emulated(a, huber, SolverOptions(max_iters=2), dev, 3)
print("sharded", rep.termination, rep.final_cost, raw.pcg_iterations)
# device-resident iterative_map: RANSAC, BA rounds, gating
sc = make_scene(24, 1500, 7500, shape="curve", seed=3, outlier_frac=0.05, depth=(2.0, 40.0))
models, n_models, fm = model_table([CameraModel(**sc.camera)] * sc.n_frames)
ptr = np.searchsorted(sc.obs_point, np.arange(sc.n_points + 1)).astype(np.int64)
F = sc.n_frames
edges = np.stack([np.arange(F - 1), np.arange(1, F)], 1).astype(np.int32)
priors = np.flatnonzero(sc.frame_fixed == 0).astype(np.int32)
r = iterative_map_arrays(sc.cam_q, sc.cam_t, fm, sc.frame_fixed, models, n_models, ptr, sc.obs_frame,
                         sc.obs_uv, edges, priors, MappingConfig(max_solver_iters=5))
print("imap", r.round_stats)
""" % REPO


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "3", sys.executable, "-c", WORKLOAD]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    with open(os.path.join(REPO, "gpurun_out", f"sanitizer_{tool}.log"), "w") as f:
        f.write(out)
    assert "imap" in out, out[-3000:]
    clean = ("RACECHECK SUMMARY: 0 hazards displayed (0 errors" if tool == "racecheck"
             else "ERROR SUMMARY: 0 errors")
    assert clean in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
