"""Parity deviation vs PCG rtol on a 1.4M-observation Venice scene (4 LM iterations)."""
import sys, numpy as np
sys.path.insert(0, '.')
from oracle import ba as OB
def oracle_problem(a):
    return OB.BAProblem(a.cam_q, a.cam_t, a.frame_model, a.frame_fixed,
                        [(0, 500.0, 500.0, 320.0, 240.0, (0.0, 0.0))], a.points, a.obs_frame,
                        a.obs_point, a.obs_uv, a.edge_ab, a.prior_frame, a.edge_weight, a.prior_weight)
from paper_2510_15271_b200.mapping import solve_arrays
from paper_2510_15271_b200.scenes import make_scene, scene_arrays
from paper_2510_15271_b200.solver import DeviceOptions, RobustLoss, SolverOptions
a = scene_arrays(make_scene(600, 300000, 1500000, shape="venice", seed=1))
qo, to, Xo, ro = oracle_problem(a).solve(1, 2.0, 4)
for rtol in (1e-12, 1e-10, 1e-8, 1e-6):
    q, t, X, rep, raw = solve_arrays(a, RobustLoss("huber", 2.0), SolverOptions(max_iters=4),
                                     DeviceOptions(linear_solver="pcg", pcg_rtol=rtol))
    sc = np.abs(Xo).max()
    print(f"rtol {rtol:.0e}: cost rel {abs(rep.final_cost-ro['final_cost'])/ro['final_cost']:.2e} "
          f"X {np.abs(X-Xo).max()/sc:.2e} t {np.abs(t-to).max()/sc:.2e} q {np.abs(q-qo).max():.2e} pcg {raw.pcg_iterations}", flush=True)
