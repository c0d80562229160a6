"""CPU study: PCG iteration counts on the config-3 reduced camera system for
preconditioner variants (block-Jacobi, the additive two-level preconditioner
the kernel uses, and deflation / A-DEF2 with the same rigid-motion coarse
space).  Builds S with the oracle's linearisation at the initial state.
usage: python tools/precond_study.py [CFG] [CLUSTER] [LAMBDA] [LM_STEPS]"""
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from oracle import ba as OB  # noqa: E402  (test infrastructure: a study, not the product)
from oracle import geometry as G  # noqa: E402
from paper_2510_15271_b200.scenes import config_scene, scene_arrays  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
C = int(sys.argv[2]) if len(sys.argv) > 2 else 12
lam = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-4
t0 = time.time()
a = scene_arrays(config_scene(cfg, seed=0), 1.0, 1.0)
pb = OB.BAProblem(a.cam_q, a.cam_t, a.frame_model, a.frame_fixed,
                  [(0, 500.0, 500.0, 320.0, 240.0, (0.0, 0.0))], a.points, a.obs_frame,
                  a.obs_point, a.obs_uv, a.edge_ab, a.prior_frame, a.edge_weight, a.prior_weight)


def build(q, t, X, lam):
    lin = pb.linearize(q, t, X, 1, 2.0)
    nf = pb.nf
    V, gp = lin["V"], lin["gp"]
    dV = np.maximum(np.einsum("pii->pi", V), 1e-12)
    Vinv = np.linalg.inv(V + lam * np.einsum("pi,ij->pij", dV, np.eye(3)))
    e = np.einsum("pij,pj->pi", Vinv, gp)
    U, gc, W, j = lin["U"], lin["gc"], lin["W"], lin["j"]
    dU = np.maximum(np.einsum("cii->ci", U), 1e-12)
    diag = U + lam * np.einsum("ci,ij->cij", dU, np.eye(6))
    keys_all, vals_all = [], []
    for (ja, jb), H in lin["Hoff"].items():
        keys_all.append(np.array([ja * nf + jb, jb * nf + ja]))
        vals_all.append(np.stack([H, H.T]))
    keys_all.append(np.arange(nf) * (nf + 1))
    vals_all.append(diag)
    pa, pbb = pb._pairs()
    CH = 1 << 19
    for s0 in range(0, len(pa), CH):
        aa, bb = pa[s0:s0 + CH], pbb[s0:s0 + CH]
        Y = np.matmul(W[aa], Vinv[pb.op[aa]])
        keys_all.append(j[aa] * nf + j[bb])
        vals_all.append(-np.matmul(Y, np.transpose(W[bb], (0, 2, 1))))
    keys = np.concatenate(keys_all)
    vals = np.concatenate(vals_all)
    uk, inv = np.unique(keys, return_inverse=True)
    blocks = np.zeros((len(uk), 6, 6))
    for r in range(6):
        for c in range(6):
            blocks[:, r, c] = np.bincount(inv, weights=vals[:, r, c], minlength=len(uk))
    rows, cols = uk // nf, uk % nf
    S = sp.bsr_matrix((blocks, cols, np.searchsorted(rows, np.arange(nf + 1))), shape=(6 * nf, 6 * nf))
    rhs = np.zeros((nf, 6))
    fr = j >= 0
    np.add.at(rhs, j[fr], np.einsum("nij,nj->ni", W[fr], e[pb.op[fr]]))
    b = (-gc + rhs).reshape(-1)
    dblocks = blocks[np.searchsorted(uk, np.arange(nf) * (nf + 1))]
    return S, b, dblocks, dict(W=W, j=j, Vinv=Vinv, e=e)


prev_dc = []  # camera steps of the previous LM iterations (warm-start study)


def step(S, b, aux, q, t, X):
    import scipy.sparse.linalg as spl
    dc = spl.spsolve(S.tocsc(), b).reshape(-1, 6)
    prev_dc.append(dc.reshape(-1).copy())
    W, j, Vinv, e = aux["W"], aux["j"], aux["Vinv"], aux["e"]
    acc = np.zeros((pb.P, 3))
    fr = j >= 0
    np.add.at(acc, pb.op[fr], np.einsum("nij,ni->nj", W[fr], dc[j[fr]]))
    dp = -e - np.einsum("pij,pj->pi", Vinv, acc)
    return pb.retract(q, t, X, dc, dp)


nlm = int(sys.argv[4]) if len(sys.argv) > 4 else 0
q, t, X = pb.q0, pb.t0, pb.X0
lam_k = lam
basis0 = None
S_hist = []
for k in range(nlm):
    S, b, dblocks, aux = build(q, t, X, lam_k)
    S_hist.append((S, q.copy(), t.copy()))
    if basis0 is None:
        basis0 = (q.copy(), t.copy(), S)
    q, t, X = step(S, b, aux, q, t, X)
    print(f"LM {k}: cost {pb.cost(q, t, X, 1, 2.0):.6e}", flush=True)
    lam_k *= 0.5
S, b, dblocks, aux = build(q, t, X, lam_k)
nf = pb.nf
print(f"S at LM {nlm} (lambda {lam_k:.2e}) built in {time.time() - t0:.1f}s", flush=True)

Dinv = np.linalg.inv(dblocks)
free = np.flatnonzero(pb.free_idx >= 0)
nc = (nf + C - 1) // C
cl = np.arange(nf) // C


def coarse(qq, tt, SS):
    Pd = np.zeros((nf, 6, 6))
    for i, f in enumerate(free):
        Pd[i] = G.adjoint(G.pose(qq[f], tt[f]))
    P = sp.bsr_matrix((Pd, cl, np.arange(nf + 1)), shape=(6 * nf, 6 * nc)).tocsr()
    return P, np.linalg.inv((P.T @ (SS @ P)).toarray())


P, Aci = coarse(q, t, S)


def jac(r):
    return np.einsum("nij,nj->ni", Dinv, r.reshape(nf, 6)).reshape(-1)


def Q(r):
    return P @ (Aci @ (P.T @ r))


def pcg(apply_m, x0, name, maxit=5000, rtol=1e-8):
    x = x0.copy()
    r = b - S @ x
    z = apply_m(r)
    p = z.copy()
    rz = r @ z
    bn = np.linalg.norm(b)
    for it in range(1, maxit + 1):
        q = S @ p
        al = rz / (p @ q)
        x += al * p
        r -= al * q
        if np.linalg.norm(r) <= rtol * bn:
            break
        z = apply_m(r)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    xs = np.linalg.norm(x)
    print(f"{name:28s} iterations {it:5d}  |r|/|b| {np.linalg.norm(b - S @ x) / bn:.2e}  |x| {xs:.6e}",
          flush=True)
    return x


zero = np.zeros_like(b)
if basis0 is not None:  # the kernel's refresh: coarse operator from LM 0
    P0, Aci0 = coarse(basis0[0], basis0[1], basis0[2])
    pcg(lambda r: jac(r) + P0 @ (Aci0 @ (P0.T @ r)), zero, f"additive, stale coarse C={C}")
pcg(jac, zero, "block-Jacobi")
pcg(lambda r: jac(r) + Q(r), zero, f"additive two-level C={C}")
# A-DEF2: M^-1 r = (I - Q S) D^-1 r + Q r, started from x0 = Q b
pcg(lambda r: (lambda z: z - Q(S @ z) + Q(r))(jac(r)), Q(b), f"A-DEF2 C={C}")
# BNN (symmetric): (I - QS) D^-1 (I - SQ) r + Q r
pcg(lambda r: (lambda z: z - Q(S @ z))(jac(r - S @ Q(r))) + Q(r), zero, f"BNN C={C}")

# --- further additive variants (same communication pattern as the kernel) ---
import os
if os.environ.get("MORE"):
    for om in (0.5, 0.75, 1.5):
        pcg(lambda r: jac(r) + om * Q(r), zero, f"additive, coarse x{om}")
    # cluster-local dense smoother (72x72 blocks) + coarse
    Sc = S.tocsr()
    Lb = []
    for c in range(nc):
        i0, i1 = 6 * c * C, min(6 * nf, 6 * (c + 1) * C)
        Lb.append(np.linalg.inv(Sc[i0:i1, i0:i1].toarray()))
    def cjac(r):
        out = np.empty_like(r)
        for c in range(nc):
            i0, i1 = 6 * c * C, min(6 * nf, 6 * (c + 1) * C)
            out[i0:i1] = Lb[c] @ r[i0:i1]
        return out
    pcg(cjac, zero, "cluster-local dense")
    pcg(lambda r: cjac(r) + Q(r), zero, "cluster-local dense + coarse")
    # symmetric multiplicative (V-cycle: Jacobi, coarse, Jacobi) -- 2 SpMV per apply
    def vcyc(r):
        z = jac(r)
        z = z + Q(r - S @ z)
        return z + jac(r - S @ z)
    pcg(vcyc, zero, "V-cycle (J, coarse, J)")

if os.environ.get("CLUSTERS"):
    for Cx in [int(v) for v in os.environ["CLUSTERS"].split(",")]:
        ncx = (nf + Cx - 1) // Cx
        clx = np.arange(nf) // Cx
        Pd = np.zeros((nf, 6, 6))
        for i, f in enumerate(free):
            Pd[i] = G.adjoint(G.pose(q[f], t[f]))
        Px = sp.bsr_matrix((Pd, clx, np.arange(nf + 1)), shape=(6 * nf, 6 * ncx)).tocsr()
        Acix = np.linalg.inv((Px.T @ (S @ Px)).toarray())
        pcg(lambda r: jac(r) + Px @ (Acix @ (Px.T @ r)), zero, f"additive two-level C={Cx} (nc={ncx})")


# --- the kernel-shaped deflated CG (next-round design, see DESIGN "Next") ---
# Per iteration, with clusters = CTAs: u = S z (own rows); t_c = P_c^T u
# (own cluster); mu = E^-1 t (E = P^T S P exact); p = z + beta p - P mu;
# q = u + beta q - (SP) mu;  pq from the recurrence formula (no extra
# reduction); alpha = rz / pq; x += alpha p; r -= alpha q; z = D^-1 r.
# Three reductions per iteration: (t, z.u, z.q_old) | (t.mu) | (r.z, r.r).
if os.environ.get("DCG"):
    E = (P.T @ (S @ P)).toarray()
    Ei = np.linalg.inv(E)
    SP = (S @ P).tocsr()

    def dcg(x0, name, maxit=5000, rtol=1e-8, formula=True):
        bn = np.linalg.norm(b)
        # x0 -> x0 + Q (b - S x0): residual orthogonal to range(P)
        x = x0 + P @ (Ei @ (P.T @ (b - S @ x0)))
        r = b - S @ x
        z = jac(r)
        p = np.zeros_like(b); q = np.zeros_like(b)
        rz = r @ z; pq_old = 1.0; beta = 0.0
        for it in range(1, maxit + 1):
            u = S @ z
            t = P.T @ u
            mu = Ei @ t
            zu, zq = z @ u, z @ q
            p = z + beta * p - P @ mu
            q = u + beta * q - SP @ mu
            pq = (zu + beta * beta * pq_old + 2 * beta * zq - t @ mu) if formula else p @ q
            al = rz / pq
            x += al * p
            r -= al * q
            if np.linalg.norm(r) <= rtol * bn:
                break
            z = jac(r)
            rz_new = r @ z
            beta = rz_new / rz
            rz = rz_new
            pq_old = pq
        true = np.linalg.norm(b - S @ x) / bn
        print(f"{name:28s} iterations {it:5d}  |r|/|b| {true:.2e}  |x| {np.linalg.norm(x):.6e}", flush=True)
    dcg(zero, "DCG, pq direct", formula=False)
    dcg(zero, "DCG, pq recurrence")


# --- warm starts: energy-optimal multiple of the previous step (the kernel)
# vs the energy-optimal combination of the previous two steps ---------------
if os.environ.get("WARM") and len(prev_dc) >= 2:
    x1, x2 = prev_dc[-1], prev_dc[-2]
    Sx1, Sx2 = S @ x1, S @ x2
    g = (x1 @ b) / (x1 @ Sx1)
    pcg(lambda r: jac(r) + Q(r), g * x1, "additive, warm gamma*x_prev")
    G2 = np.array([[x1 @ Sx1, x1 @ Sx2], [x2 @ Sx1, x2 @ Sx2]])
    c = np.linalg.solve(G2, np.array([x1 @ b, x2 @ b]))
    pcg(lambda r: jac(r) + Q(r), c[0] * x1 + c[1] * x2, "additive, warm 2-vector")
    if len(prev_dc) >= 3:
        x3 = prev_dc[-3]
        V = np.stack([x1, x2, x3], 1)
        SV = np.stack([Sx1, Sx2, S @ x3], 1)
        c3 = np.linalg.solve(V.T @ SV, V.T @ b)
        pcg(lambda r: jac(r) + Q(r), V @ c3, "additive, warm 3-vector")


# --- Newton-Schulz refresh of the coarse inverse: how far is the previous
# solve's exact inverse from the new one?  eps0 = ||I - E_new X_old||_2 ----
if os.environ.get("NS") and S_hist:
    P_new, Aci_new = coarse(q, t, S)
    E_new = (P_new.T @ (S @ P_new)).toarray()
    Sp, qp, tp = S_hist[-1]
    P_old, X_old = coarse(qp, tp, Sp)
    I = np.eye(E_new.shape[0])
    e0 = np.linalg.norm(I - E_new @ X_old, 2)
    print(f"NS: eps0 (previous LM iteration, new basis) = {e0:.3e}", flush=True)
    X = X_old.copy()
    for it in range(4):
        X = X @ (2 * I - E_new @ X)
        print(f"NS step {it + 1}: ||I - E X|| = {np.linalg.norm(I - E_new @ X, 2):.3e}", flush=True)


# --- coarse space + a per-cluster scale column: the similarity gauge's scale
# direction of camera j is the left perturbation (0, t_j) (t -> s t), which
# the rigid-motion columns Adj(T_j) do not span ------------------------------
if os.environ.get("SCALE"):
    for Cx in [int(v) for v in os.environ.get("SCALE_C", str(C)).split(",")]:
        # balanced clusters of ~Cx frames (no one-frame tail: 7 columns need 2+ frames)
        ncx = max(1, nf // Cx)
        clx = (np.arange(nf) * ncx) // nf
        Pd = np.zeros((nf, 6, 7))
        for i, f in enumerate(free):
            qq, tt = G.pose(q[f], t[f])
            Pd[i, :, :6] = G.adjoint((qq, tt))
            Pd[i, 3:, 6] = tt
        Px = sp.bsr_matrix((Pd, clx, np.arange(nf + 1)), shape=(6 * nf, 7 * ncx)).tocsr()
        Ax = (Px.T @ (S @ Px)).toarray()
        ev = np.linalg.eigvalsh(Ax)
        print(f"rigid+scale C={Cx}: A_c eigenvalues {ev[0]:.3e} .. {ev[-1]:.3e}", flush=True)
        Acix = np.linalg.inv(Ax)
        pcg(lambda r: jac(r) + Px @ (Acix @ (Px.T @ r)), zero, f"additive rigid+scale C={Cx}")
        # the same space with each cluster's 7 columns orthonormalised first
        # (QR of the cluster's stacked 6n x 7 block): same span, A_c well scaled
        Pq = np.zeros_like(Pd)
        for c in range(ncx):
            rows = np.flatnonzero(clx == c)
            Bc = Pd[rows].reshape(-1, 7)
            Q, _ = np.linalg.qr(Bc)
            Pq[rows] = Q.reshape(len(rows), 6, 7)
        Pxq = sp.bsr_matrix((Pq, clx, np.arange(nf + 1)), shape=(6 * nf, 7 * ncx)).tocsr()
        Aq = (Pxq.T @ (S @ Pxq)).toarray()
        evq = np.linalg.eigvalsh(Aq)
        print(f"rigid+scale C={Cx} orthonormal: A_c eigenvalues {evq[0]:.3e} .. {evq[-1]:.3e}", flush=True)
        Aciq = np.linalg.inv(Aq)
        pcg(lambda r: jac(r) + Pxq @ (Aciq @ (Pxq.T @ r)), zero, f"additive rigid+scale C={Cx} orthonormal")
        # rigid only, orthonormalised (the same span as the kernel's)
        Pr = np.zeros((nf, 6, 6))
        for c in range(ncx):
            rows = np.flatnonzero(clx == c)
            Q, _ = np.linalg.qr(Pd[rows, :, :6].reshape(-1, 6))
            Pr[rows] = Q.reshape(len(rows), 6, 6)
        Pxr = sp.bsr_matrix((Pr, clx, np.arange(nf + 1)), shape=(6 * nf, 6 * ncx)).tocsr()
        Acir = np.linalg.inv((Pxr.T @ (S @ Pxr)).toarray())
        pcg(lambda r: jac(r) + Pxr @ (Acir @ (Pxr.T @ r)), zero, f"additive rigid C={Cx} orthonormal")
        # global similarity (7 columns over all frames) on top of the rigid clusters
    Pg = np.zeros((nf, 6, 7))
    for i, f in enumerate(free):
        qq, tt = G.pose(q[f], t[f])
        Pg[i, :, :6] = G.adjoint((qq, tt))
        Pg[i, 3:, 6] = tt
    Pg = Pg.reshape(6 * nf, 7)
    Pfull = sp.hstack([P, sp.csr_matrix(Pg)]).tocsr()
    Acif = np.linalg.pinv((Pfull.T @ (S @ Pfull)).toarray())
    pcg(lambda r: jac(r) + Pfull @ (Acif @ (Pfull.T @ r)), zero, f"additive rigid C={C} + global similarity")
