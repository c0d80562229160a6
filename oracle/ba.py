"""numpy restatement of the reference LM bundle adjustment (oracle only).

Follows solver.solve (solver.py:194-257) as driven by bundle_adjust
(mapping.py:390-527) on the flattened layout of include/sfm_b200.h:

  * residuals: reprojection per observation (robust loss, mapping.py:452-475),
    lambda_c sequential edges (posegraph.py:195-206, measurement taken from
    the entry poses, mapping.py:477-498), lambda_a absolute priors
    (mapping.py:359-368, :500-509); cost = sum rho(|r|^2), no 1/2
    (solver.py:132-151), summed sequentially in residual order;
  * IRLS weighting sqrt(rho'(s)) on r and J (solver.py:170-178);
  * Marquardt damping D = max(diag H, 1e-12) over all free parameters
    (solver.py:217), lambda schedule 1e-4 / x10 / x0.5 floor 1e-18 / cap
    1e32, rejected trials reuse H and g (solver.py:206-245);
  * termination rules and SolverReport fields (solver.py:209-257).

The normal equations are solved exactly through the Schur complement on the
cameras and a dense Cholesky (scipy) instead of SuperLU on the un-reduced
system (solver.py:222) -- the same linear system, solved to rounding.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

from . import geometry as G

TERMINATIONS = ("max_iterations", "gradient_tolerance", "no_decrease",
                "parameter_tolerance", "cost_zero", "all_fixed")


class OracleNonPositiveDepth(Exception):
    """NonPositiveDepth raised while evaluating a cost (cameras.py:132-133)."""


class OracleSolverDiverged(Exception):
    """SolverDiverged (solver.py:247-248)."""


class BAProblem:
    """Flattened problem (same fields as sfm_ba_problem)."""

    def __init__(self, cam_q, cam_t, frame_model, frame_fixed, models, points, obs_frame,
                 obs_point, obs_uv, edge_ab=None, prior_frame=None, edge_weight=0.0,
                 prior_weight=0.0):
        self.q0 = np.asarray(cam_q, float).reshape(-1, 4)
        self.t0 = np.asarray(cam_t, float).reshape(-1, 3)
        self.fm = np.asarray(frame_model, np.int64)
        self.fixed = np.asarray(frame_fixed, bool)
        self.models = list(models)
        self.X0 = np.asarray(points, float).reshape(-1, 3)
        self.of = np.asarray(obs_frame, np.int64)
        self.op = np.asarray(obs_point, np.int64)
        self.uv = np.asarray(obs_uv, float).reshape(-1, 2)
        self.edges = np.zeros((0, 2), np.int64) if edge_ab is None else \
            np.asarray(edge_ab, np.int64).reshape(-1, 2)
        self.priors = np.zeros(0, np.int64) if prior_frame is None else \
            np.asarray(prior_frame, np.int64)
        self.we = np.sqrt(edge_weight)   # information_sqrt(lambda_c I) = sqrt(lambda_c) I
        self.wa = np.sqrt(prior_weight)
        F = len(self.q0)
        self.free_idx = np.full(F, -1, np.int64)
        free = np.flatnonzero(~self.fixed)
        self.free_idx[free] = np.arange(len(free))
        self.nf = len(free)
        self.P = len(self.X0)
        self.N = len(self.of)
        # pose-term constants from the entry poses
        entry = [G.pose(self.q0[f], self.t0[f]) for f in range(F)]
        self.meas_inv = [G.pinv(G.pmul(entry[a], G.pinv(entry[b]))) for a, b in self.edges]
        self.adj_meas_inv = [G.adjoint(m) for m in self.meas_inv]
        self.init_inv = [G.pinv(entry[f]) for f in self.priors]

    # --- residuals ------------------------------------------------------
    def _cams(self, q, t):
        return G.qmat(q), t

    def obs_project(self, q, t, X, jac=False, idx=None):
        """Raw reprojection residual pix - uv per observation (+ Jacobians)."""
        of = self.of if idx is None else self.of[idx]
        op = self.op if idx is None else self.op[idx]
        uv = self.uv if idx is None else self.uv[idx]
        R = G.qmat(q)
        n = len(of)
        r = np.zeros((n, 2))
        st = np.zeros(n, np.int8)
        Jc = np.zeros((n, 2, 6)) if jac else None
        Jp = np.zeros((n, 2, 3)) if jac else None
        for m in np.unique(self.fm[of]) if n else []:
            sel = np.flatnonzero(self.fm[of] == m)
            model = self.models[m]
            Rs, ts, Xs = R[of[sel]], t[of[sel]], X[op[sel]]
            if jac:
                pix, jc, jp, s = G.project_with_jacobians(model, Rs, ts, Xs)
                Jc[sel], Jp[sel] = jc, jp
            else:
                pc = np.einsum("nij,nj->ni", Rs, Xs) + ts
                pix, s = G.project_cam(model, pc)
            r[sel] = pix - uv[sel]
            st[sel] = s
        return r, st, Jc, Jp

    def edge_terms(self, q, t, jac=False):
        out = []
        for e, (a, b) in enumerate(self.edges):
            Ta, Tb = G.pose(q[a], t[a]), G.pose(q[b], t[b])
            rr = G.log_map(G.pmul(G.pmul(self.meas_inv[e], Ta), G.pinv(Tb)))
            if jac:
                Ja = self.we * (G.se3_jl_inv(rr) @ self.adj_meas_inv[e])
                Jb = self.we * (-G.se3_jl_inv(-rr))
                out.append((self.we * rr, Ja, Jb))
            else:
                out.append(self.we * rr)
        return out

    def prior_terms(self, q, t, jac=False):
        out = []
        for k, f in enumerate(self.priors):
            rr = G.log_map(G.pmul(G.pose(q[f], t[f]), self.init_inv[k]))
            out.append((self.wa * rr, self.wa * G.se3_jl_inv(rr)) if jac else self.wa * rr)
        return out

    def cost(self, q, t, X, loss_kind, loss_param):
        """Problem.evaluate / _cost_only (solver.py:132-151)."""
        r, st, _, _ = self.obs_project(q, t, X)
        bad = np.flatnonzero(st != G.OK)
        if len(bad):
            o = bad[0]
            pc = G.qmat(q[self.of[o]]) @ X[self.op[o]] + t[self.of[o]]
            raise OracleNonPositiveDepth(f"depth {pc[2]:.3e}")
        s = r[:, 0] * r[:, 0] + r[:, 1] * r[:, 1]
        parts = [G.loss_rho(loss_kind, loss_param, s)]
        parts.append(np.array([float(v @ v) for v in self.edge_terms(q, t)]))
        parts.append(np.array([float(v @ v) for v in self.prior_terms(q, t)]))
        allv = np.concatenate(parts)
        return float(np.cumsum(allv)[-1]) if len(allv) else 0.0

    # --- linearisation (solver.py:164-191, 210-217) ---------------------
    def linearize(self, q, t, X, loss_kind, loss_param):
        r, st, Jc, Jp = self.obs_project(q, t, X, jac=True)
        s = r[:, 0] * r[:, 0] + r[:, 1] * r[:, 1]
        w = np.sqrt(G.loss_rho_prime(loss_kind, loss_param, s))
        rt = r * w[:, None]
        Jc = Jc * w[:, None, None]
        Jp = Jp * w[:, None, None]
        nf, P = self.nf, self.P
        V = np.zeros((P, 3, 3))
        gp = np.zeros((P, 3))
        np.add.at(V, self.op, np.einsum("nki,nkj->nij", Jp, Jp))
        np.add.at(gp, self.op, np.einsum("nki,nk->ni", Jp, rt))
        U = np.zeros((nf, 6, 6))
        gc = np.zeros((nf, 6))
        j = self.free_idx[self.of]
        fr = j >= 0
        np.add.at(U, j[fr], np.einsum("nki,nkj->nij", Jc[fr], Jc[fr]))
        np.add.at(gc, j[fr], np.einsum("nki,nk->ni", Jc[fr], rt[fr]))
        W = np.einsum("nki,nkj->nij", Jc, Jp)  # [N,6,3]
        Hoff = {}
        for e, ((a, b), (re, Ja, Jb)) in enumerate(zip(self.edges, self.edge_terms(q, t, True))):
            ja, jb = self.free_idx[a], self.free_idx[b]
            if ja >= 0:
                U[ja] += Ja.T @ Ja
                gc[ja] += Ja.T @ re
            if jb >= 0:
                U[jb] += Jb.T @ Jb
                gc[jb] += Jb.T @ re
            if ja >= 0 and jb >= 0:
                Hoff[(ja, jb)] = Hoff.get((ja, jb), 0.0) + Ja.T @ Jb
        for f, (rp, J) in zip(self.priors, self.prior_terms(q, t, True)):
            jf = self.free_idx[f]
            if jf >= 0:
                U[jf] += J.T @ J
                gc[jf] += J.T @ rp
        return dict(V=V, gp=gp, U=U, gc=gc, W=W, j=j, Hoff=Hoff, Jc=Jc, Jp=Jp, rt=rt)

    def _pairs(self):
        if hasattr(self, "_pair_cache"):
            return self._pair_cache
        k = np.bincount(self.op, minlength=self.P)
        start = np.concatenate([[0], np.cumsum(k)[:-1]])
        kk = k[self.op]
        a = np.repeat(np.arange(self.N), kk)
        first = np.repeat(np.cumsum(kk) - kk, kk)
        b = np.repeat(start[self.op], kk) + (np.arange(len(a)) - first)
        j = self.free_idx[self.of]
        keep = (j[a] >= 0) & (j[b] >= 0)
        self._pair_cache = (a[keep], b[keep])
        return self._pair_cache

    def reduced_system(self, lin, lam):
        """S = U* - sum W V*^-1 W^T, b = -g_c + sum W V*^-1 g_p (dense)."""
        V, gp = lin["V"], lin["gp"]
        dV = np.maximum(np.einsum("pii->pi", V), 1e-12)
        Vs = V + lam * np.einsum("pi,ij->pij", dV, np.eye(3))
        Vinv = np.linalg.inv(Vs)
        e = np.einsum("pij,pj->pi", Vinv, gp)
        nf = self.nf
        U, gc, W, j = lin["U"], lin["gc"], lin["W"], lin["j"]
        dU = np.maximum(np.einsum("cii->ci", U), 1e-12)
        S4 = np.zeros((nf, nf, 6, 6))
        S4[np.arange(nf), np.arange(nf)] = U + lam * np.einsum("ci,ij->cij", dU, np.eye(6))
        for (ja, jb), H in lin["Hoff"].items():
            S4[ja, jb] += H
            S4[jb, ja] += H.T
        S_pt, b_pt = self.point_schur_terms(lin, Vinv, e)
        S = S4.transpose(0, 2, 1, 3).reshape(6 * nf, 6 * nf) + S_pt
        return S, -gc.reshape(-1) + b_pt, Vinv, e, dV, dU

    def point_schur_terms(self, lin, Vinv, e):
        """The points' share of the reduced system: -sum_i W V*_i^-1 W^T and
        sum_i W e_i.  Under point sharding each rank holds only its points'
        share; the camera blocks are added once.  Pair
        products are batched matmuls, summed per S block with bincount (a
        different summation order than a sequential np.add.at: rounding-level
        differences only)."""
        nf, W, j = self.nf, lin["W"], lin["j"]
        a, b = self._pairs()
        key = j[a] * nf + j[b]
        acc = np.zeros((36, nf * nf))
        CH = 1 << 20
        for s0 in range(0, len(a), CH):
            aa, bb, kk = a[s0:s0 + CH], b[s0:s0 + CH], key[s0:s0 + CH]
            T = np.matmul(W[aa], Vinv[self.op[aa]])
            C = np.matmul(T, np.transpose(W[bb], (0, 2, 1))).reshape(-1, 36)
            for q in range(36):
                acc[q] -= np.bincount(kk, weights=C[:, q], minlength=nf * nf)
        S4 = acc.T.reshape(nf, nf, 6, 6)
        rhs = np.zeros((nf, 6))
        fr = j >= 0
        np.add.at(rhs, j[fr], np.einsum("nij,nj->ni", W[fr], e[self.op[fr]]))
        return S4.transpose(0, 2, 1, 3).reshape(6 * nf, 6 * nf), rhs.reshape(-1)

    def damped_points(self, lin, lam):
        """V* = V + lam max(diag V, 1e-12) (solver.py:217-220), V*^-1, e."""
        V, gp = lin["V"], lin["gp"]
        dV = np.maximum(np.einsum("pii->pi", V), 1e-12)
        Vinv = np.linalg.inv(V + lam * np.einsum("pi,ij->pij", dV, np.eye(3)))
        return Vinv, np.einsum("pij,pj->pi", Vinv, gp)

    def solve_step(self, lin, lam):
        """(H + lam D) delta = -g via the Schur complement -> (dc, dp) or None."""
        S, rhs, Vinv, e, _, _ = self.reduced_system(lin, lam)
        if self.nf:
            try:
                c = scipy.linalg.cho_factor(S, lower=True, check_finite=True)
                dc = scipy.linalg.cho_solve(c, rhs).reshape(self.nf, 6)
            except (np.linalg.LinAlgError, ValueError):
                return None
        else:
            dc = np.zeros((0, 6))
        j = lin["j"]
        acc = np.zeros((self.P, 3))
        fr = j >= 0
        np.add.at(acc, self.op[fr], np.einsum("nij,ni->nj", lin["W"][fr], dc[j[fr]]))
        dp = -e - np.einsum("pij,pj->pi", Vinv, acc)
        if not (np.all(np.isfinite(dc)) and np.all(np.isfinite(dp))):
            return None
        return dc, dp

    def retract(self, q, t, X, dc, dp):
        """ParameterBlock.retracted (solver.py:68-71)."""
        q2, t2 = q.copy(), t.copy()
        for f in np.flatnonzero(self.free_idx >= 0):
            nq, nt = G.pmul(G.exp_map(dc[self.free_idx[f]]), G.pose(q[f], t[f]))
            q2[f], t2[f] = nq, nt
        return q2, t2, X + dp

    # --- LM (solver.py:194-257) ------------------------------------------
    def solve(self, loss_kind=0, loss_param=1.0, max_iters=50, grad_tol=1e-10,
              param_tol=1e-12, initial_lambda=1e-4, max_lambda=1e32, trace=None):
        q, t, X = self.q0.copy(), self.t0.copy(), self.X0.copy()
        n_params = 6 * self.nf + 3 * self.P
        initial = self.cost(q, t, X, loss_kind, loss_param)
        has_res = self.N + len(self.edges) + len(self.priors) > 0
        if n_params == 0 or not has_res:
            return q, t, X, dict(initial_cost=initial, final_cost=initial, iterations=0,
                                 termination="all_fixed")
        cost, lam, iters, term = initial, initial_lambda, 0, "max_iterations"
        for iters in range(1, max_iters + 1):
            lin = self.linearize(q, t, X, loss_kind, loss_param)
            g = np.concatenate([lin["gc"].ravel(), lin["gp"].ravel()])
            if np.max(np.abs(g)) < grad_tol:
                term = "gradient_tolerance"
                iters -= 1
                break
            accepted = False
            while lam <= max_lambda:
                step = self.solve_step(lin, lam)
                if step is None:
                    lam *= 10.0
                    continue
                dc, dp = step
                qn, tn, Xn = self.retract(q, t, X, dc, dp)
                new_cost = self.cost(qn, tn, Xn, loss_kind, loss_param)
                if trace is not None:
                    trace.append((iters, lam, new_cost))
                if np.isfinite(new_cost) and new_cost < cost:
                    q, t, X = qn, tn, Xn
                    step_norm = float(np.sqrt(np.sum(dc * dc) + np.sum(dp * dp)))
                    cost = new_cost
                    lam = max(lam * 0.5, 1e-18)
                    accepted = True
                    break
                lam *= 10.0
            if not accepted:
                if lam > max_lambda and cost > initial:
                    raise OracleSolverDiverged(f"damping overflow at cost {cost}")
                term = "no_decrease"
                break
            if step_norm < param_tol * (np.sqrt(n_params) + param_tol):
                term = "parameter_tolerance"
                break
            if cost < 1e-30:
                term = "cost_zero"
                break
        return q, t, X, dict(initial_cost=initial, final_cost=cost, iterations=iters,
                             termination=term)


def problem_from_npz(d, prefix=""):
    """Builds a BAProblem from golden-fixture arrays."""
    models = [(int(k), float(fx), float(fy), float(cx), float(cy), (float(k1), float(k2)))
              for k, fx, fy, cx, cy, k1, k2 in np.asarray(d[prefix + "models"]).reshape(-1, 7)]
    return BAProblem(d[prefix + "cam_q"], d[prefix + "cam_t"], d[prefix + "frame_model"],
                     d[prefix + "frame_fixed"], models, d[prefix + "points"],
                     d[prefix + "obs_frame"], d[prefix + "obs_point"], d[prefix + "obs_uv"],
                     d[prefix + "edge_ab"], d[prefix + "prior_frame"],
                     float(d[prefix + "edge_weight"]), float(d[prefix + "prior_weight"]))
