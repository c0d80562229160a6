"""Golden LM trajectory of the benchmarked configuration (BASELINE.json
configs[2], the bench.py workload): the pinned CPU oracle (oracle/ba.py, a
restatement of solver.solve, solver.py:194-257, checked against sfmkit's own
outputs in tests/test_oracle_golden.py) runs the config-3 scene (seed 0,
Huber delta 2, lambda_c = lambda_a = 1, the stage-1 defaults of
mapping.py:92-96) from its initial state to LM termination with an exact
Schur + dense Cholesky solve of every damped system.

Stored (tests/golden/config3_lm.npz):
  trace_it, trace_lam, trace_cost   every trial (iteration, lambda, trial cost)
  costs                             accepted cost after each iteration
  initial_cost, final_cost, iterations, termination
  cam_q, cam_t                      final poses (all 1,778 frames)
  pt_idx, pt_sample                 final positions of a fixed point sample
  pt_mean, pt_absmean               mean / mean |x| of all final positions

Run on a CPU box (about an hour with 8 threads); the GPU test
tests/test_gpu_configs.py::test_config3_lm_to_termination_matches_oracle
compares the device solve against it.

    python tests/golden/make_config3_lm.py [out.npz]
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)


def main(out):
    from oracle import ba as OB
    from paper_2510_15271_b200.scenes import config_scene, scene_arrays

    t0 = time.time()
    sc = config_scene(3, seed=0)
    a = scene_arrays(sc, lambda_c=1.0, lambda_a=1.0)
    models = [(0, 500.0, 500.0, 320.0, 240.0, (0.0, 0.0))]
    prob = OB.BAProblem(a.cam_q, a.cam_t, a.frame_model, a.frame_fixed, models, a.points,
                        a.obs_frame, a.obs_point, a.obs_uv, a.edge_ab, a.prior_frame,
                        a.edge_weight, a.prior_weight)
    print(f"scene: {sc.n_frames} frames, {sc.n_points} points, {sc.n_obs} obs "
          f"({time.time() - t0:.1f} s)", flush=True)
    trace = []

    class Tr(list):
        def append(self, x):
            super().append(x)
            it, lam, c = x
            print(f"  it {it:3d} lam {lam:.3e} cost {c!r} ({time.time() - t0:.0f} s)", flush=True)

    trace = Tr()
    q, t, X, rep = prob.solve(1, 2.0, 50, trace=trace)
    it = np.array([x[0] for x in trace], np.int32)
    lam = np.array([x[1] for x in trace])
    cost = np.array([x[2] for x in trace])
    # accepted cost per iteration: the last trial of each iteration that decreased it
    costs = []
    cur = rep["initial_cost"]
    for k in range(1, int(it.max()) + 1 if len(it) else 1):
        sel = np.flatnonzero(it == k)
        acc = [c for c in cost[sel] if np.isfinite(c) and c < cur]
        if acc:
            cur = acc[-1]
            costs.append(cur)
    rng = np.random.default_rng(12345)
    pt_idx = np.sort(rng.choice(len(X), size=2000, replace=False))
    np.savez_compressed(out, trace_it=it, trace_lam=lam, trace_cost=cost, costs=np.array(costs),
                        initial_cost=rep["initial_cost"], final_cost=rep["final_cost"],
                        iterations=rep["iterations"], termination=rep["termination"],
                        cam_q=q, cam_t=t, pt_idx=pt_idx, pt_sample=X[pt_idx],
                        pt_mean=X.mean(0), pt_absmean=np.abs(X).mean(0),
                        n_frames=sc.n_frames, n_points=sc.n_points, n_obs=sc.n_obs)
    print(f"done: {rep} in {time.time() - t0:.0f} s -> {out}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "config3_lm.npz"))
