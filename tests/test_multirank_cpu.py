"""World-size-2 CPU (gloo) tests of the point-sharded multi-GPU path
(SURVEY.md §8(e)): the host-side sharding, the camera-indexed reductions
that csrc/comm.cuh performs with NCCL, and the gather of the sharded points.

Each rank takes its shard (`BAArrays.shard`, boundaries checked against the
library's own host-side split, sfm_shard_points), computes its partial
linearisation / reduced camera system with the oracle, and the partials are
all-reduced over gloo, exactly where libsfm_b200 all-reduces over NCCL
(linearize(): U, g_c, grad max; build_schur(): S, b_S; trial(): cost).  The
sum must equal the unsharded system.  The row-partitioned variant is then
replayed with the library's rank row ranges (sfm_pcg_rank_rows): S and b
reduce-scattered by block rows, a CG in which every rank updates only its
rows, exchanging z (all_gather) and the dot products (all_reduce) each
iteration, the solution allgathered -- and it equals the unsharded step.  No
GPU is needed (the two helpers are host-only).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    from paper_2510_15271_b200.scenes import make_scene, scene_arrays
    sc = make_scene(10, 400, 2000, shape="venice", seed=11)
    return scene_arrays(sc)


def _oracle(a):
    from oracle import ba as OB
    return OB.BAProblem(a.cam_q, a.cam_t, a.frame_model, a.frame_fixed,
                        [(0, 500.0, 500.0, 320.0, 240.0, (0.0, 0.0))], a.points, a.obs_frame,
                        a.obs_point, a.obs_uv, a.edge_ab, a.prior_frame, a.edge_weight,
                        a.prior_weight)


def allsum_off(lin, world, dist, nf):
    """The off-diagonal pose-term blocks (rank 0's; empty elsewhere)."""
    return lin["Hoff"]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = _scene()
        part = full.shard(rank, world)
        p = _oracle(part)
        q, t, X = part.cam_q, part.cam_t, part.points
        lam = 1e-3

        def allsum(arr):
            ten = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
            dist.all_reduce(ten)
            return ten.numpy()

        # trial cost (k_finalize partials -> comm sum of cost)
        cost = allsum(np.array([p.cost(q, t, X, 1, 2.0)]))[0]
        # linearize(): U, g_c summed over ranks (pose terms live on rank 0)
        lin = p.linearize(q, t, X, 1, 2.0)
        U = allsum(lin["U"])
        gc = allsum(lin["gc"])
        # build_schur(): each rank's points' share of S and b_S, camera
        # blocks (damped with the GLOBAL diagonal) added on rank 0 only
        Vinv, e = p.damped_points(lin, lam)
        S_pt, b_pt = p.point_schur_terms(lin, Vinv, e)
        S = allsum(S_pt)
        b = allsum(b_pt)
        # _solve_sharded: gather of the sharded points in rank order
        gathered = [None] * world
        dist.all_gather_object(gathered, X)
        # row-partitioned solve (pcg_partition): the full camera blocks on
        # rank 0, the library's rank row ranges over the S block pattern
        from paper_2510_15271_b200 import _native as nat
        nf = p.nf
        S4 = np.zeros((nf, nf, 6, 6))
        if rank == 0:
            dU = np.maximum(np.einsum("cii->ci", U), 1e-12)
            S4[np.arange(nf), np.arange(nf)] = U + lam * np.einsum("ci,ij->cij", dU, np.eye(6))
            for (ja, jb), H in allsum_off(lin, world, dist, nf).items():
                S4[ja, jb] += H
                S4[jb, ja] += H.T
        else:
            allsum_off(lin, world, dist, nf)
        S_pt, b_pt = p.point_schur_terms(lin, Vinv, e)   # this rank's partials (allsum above summed in place)
        Sp = S4.transpose(0, 2, 1, 3).reshape(6 * nf, 6 * nf) + S_pt
        bp = (-gc.reshape(-1) if rank == 0 else np.zeros(6 * nf)) + b_pt
        blk_nz = np.abs(allsum(Sp.copy())).reshape(nf, 6, nf, 6).max(axis=(1, 3)) > 0
        row_ptr = np.concatenate([[0], np.cumsum(blk_nz.sum(1))]).astype(np.int32)
        rows = nat.pcg_rank_rows(row_ptr, world)
        lo, hi = 6 * rows[rank], 6 * rows[rank + 1]
        # reduce-scatter by block rows: rank r keeps the summed rows it owns
        S_own, b_own = None, None
        for q in range(world):
            a0, a1 = 6 * rows[q], 6 * rows[q + 1]
            tS = torch.from_numpy(np.ascontiguousarray(Sp[a0:a1]))
            tb = torch.from_numpy(np.ascontiguousarray(bp[a0:a1]))
            dist.reduce(tS, dst=q)
            dist.reduce(tb, dst=q)
            if q == rank:
                S_own, b_own = tS.numpy().copy(), tb.numpy().copy()
        # CG with block-Jacobi, each rank updating its rows only
        Minv = np.zeros((hi - lo, hi - lo))
        for i in range(0, hi - lo, 6):
            Minv[i:i + 6, i:i + 6] = np.linalg.inv(S_own[i:i + 6, lo + i:lo + i + 6])

        width = 6 * int(np.max(np.diff(rows)))

        def gather_vec(v):
            # allgather with variable counts (gloo wants equal sizes: pad)
            buf = np.zeros(width)
            buf[:len(v)] = v
            parts = [torch.zeros(width, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(buf))
            return np.concatenate([parts[q].numpy()[:6 * (rows[q + 1] - rows[q])] for q in range(world)])

        def dot(u, v):
            return float(allsum(np.array([u @ v]))[0])

        x = np.zeros(hi - lo)
        r_ = b_own.copy()
        z = Minv @ r_
        pv = z.copy()
        rz = dot(r_, z)
        bn = np.sqrt(dot(b_own, b_own))
        for _ in range(500):
            q_ = S_own @ gather_vec(pv)
            alpha = rz / dot(pv, q_)
            x += alpha * pv
            r_ -= alpha * q_
            if np.sqrt(dot(r_, r_)) <= 1e-13 * bn:
                break
            z = Minv @ r_
            rz_new = dot(r_, z)
            pv = z + (rz_new / rz) * pv
            rz = rz_new
        dc_part = gather_vec(x)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), cost=cost, U=U, gc=gc, S=S, b=b,
                 X=np.concatenate(gathered, axis=0), n_edges=len(part.edge_ab),
                 n_priors=len(part.prior_frame), n_obs=len(part.obs_frame),
                 obs_offset=part.obs_offset, n_params=part.n_params_global, dc_part=dc_part,
                 rank_rows=rows)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def sharded(tmp_path_factory):
    import torch.multiprocessing as mp
    out = str(tmp_path_factory.mktemp("gloo"))
    mp.start_processes(_worker, args=(WORLD, _free_port(), out), nprocs=WORLD,
                       start_method="spawn", join=True)
    return [dict(np.load(os.path.join(out, f"rank{r}.npz"))) for r in range(WORLD)]


def test_ranks_agree_bitwise(sharded):
    """An all-reduce leaves identical values on every rank, so the
    replicated PCG takes identical decisions everywhere."""
    for k in ("cost", "U", "gc", "S", "b", "X"):
        assert sharded[0][k].tobytes() == sharded[1][k].tobytes(), k


def test_shards_partition_observations_and_terms(sharded):
    full = _scene()
    assert sum(int(r["n_obs"]) for r in sharded) == len(full.obs_frame)
    assert int(sharded[0]["obs_offset"]) == 0
    assert int(sharded[1]["obs_offset"]) == int(sharded[0]["n_obs"])
    assert int(sharded[0]["n_edges"]) == len(full.edge_ab)
    assert int(sharded[1]["n_edges"]) == 0 and int(sharded[1]["n_priors"]) == 0
    n_free = int((full.frame_fixed == 0).sum())
    assert int(sharded[0]["n_params"]) == 6 * n_free + 3 * len(full.points)


def test_gathered_points_in_map_order(sharded):
    full = _scene()
    assert sharded[0]["X"].tobytes() == np.ascontiguousarray(full.points).tobytes()


def test_sharded_sums_equal_unsharded_system(sharded):
    full = _scene()
    p = _oracle(full)
    q, t, X = full.cam_q, full.cam_t, full.points
    lam = 1e-3
    r = sharded[0]
    assert r["cost"] == pytest.approx(p.cost(q, t, X, 1, 2.0), rel=1e-13)
    lin = p.linearize(q, t, X, 1, 2.0)
    np.testing.assert_allclose(r["U"], lin["U"], rtol=1e-11, atol=1e-9 * np.abs(lin["U"]).max())
    np.testing.assert_allclose(r["gc"], lin["gc"], rtol=1e-11, atol=1e-9 * np.abs(lin["gc"]).max())
    S_ref, b_ref, *_ = p.reduced_system(lin, lam)
    # rank 0 adds the camera blocks damped with the summed diagonal
    nf = p.nf
    dU = np.maximum(np.einsum("cii->ci", r["U"]), 1e-12)
    S4 = np.zeros((nf, nf, 6, 6))
    S4[np.arange(nf), np.arange(nf)] = r["U"] + lam * np.einsum("ci,ij->cij", dU, np.eye(6))
    for (ja, jb), H in lin["Hoff"].items():
        S4[ja, jb] += H
        S4[jb, ja] += H.T
    S = S4.transpose(0, 2, 1, 3).reshape(6 * nf, 6 * nf) + r["S"]
    b = -r["gc"].reshape(-1) + r["b"]
    scale = np.abs(S_ref).max()
    np.testing.assert_allclose(S, S_ref, rtol=1e-10, atol=1e-11 * scale)
    np.testing.assert_allclose(b, b_ref, rtol=1e-10, atol=1e-11 * np.abs(b_ref).max())
    # and the step it produces matches the unsharded step
    import scipy.linalg
    dc = scipy.linalg.cho_solve(scipy.linalg.cho_factor(S, lower=True), b)
    dc_ref = scipy.linalg.cho_solve(scipy.linalg.cho_factor(S_ref, lower=True), b_ref)
    np.testing.assert_allclose(dc, dc_ref, rtol=1e-8, atol=1e-10 * np.abs(dc_ref).max())


def test_library_point_shards_match_host_split():
    """sfm_shard_points (the split libsfm_b200 uses for a multi-device
    context) == mapping.shard_ranges (BAArrays.shard), and every point's
    observations stay on one rank."""
    from paper_2510_15271_b200 import _native as nat
    from paper_2510_15271_b200.mapping import shard_ranges
    from paper_2510_15271_b200.scenes import make_scene
    sc = make_scene(40, 3000, 15000, shape="venice", seed=4)
    for world in (1, 2, 3, 5, 8):
        b = nat.shard_points(sc.obs_point, sc.n_points, world)
        ref = shard_ranges(sc.obs_point, sc.n_points, world)
        assert [(int(b[r]), int(b[r + 1])) for r in range(world)] == [tuple(map(int, x)) for x in ref]
        assert b[0] == 0 and b[-1] == sc.n_points and np.all(np.diff(b) >= 0)


def test_row_partitioned_solve_equals_unsharded(sharded):
    """The replayed row-partitioned PCG data flow (reduce-scatter by the
    library's rank rows, per-rank row updates, z allgather, dot-product
    allreduce, solution allgather) gives the unsharded step, identically on
    both ranks."""
    import scipy.linalg
    full = _scene()
    p = _oracle(full)
    lin = p.linearize(full.cam_q, full.cam_t, full.points, 1, 2.0)
    S_ref, b_ref, *_ = p.reduced_system(lin, 1e-3)
    dc_ref = scipy.linalg.cho_solve(scipy.linalg.cho_factor(S_ref, lower=True), b_ref)
    assert sharded[0]["dc_part"].tobytes() == sharded[1]["dc_part"].tobytes()
    rows = sharded[0]["rank_rows"]
    assert rows[0] == 0 and rows[-1] == p.nf and np.all(np.diff(rows) >= 1)
    np.testing.assert_allclose(sharded[0]["dc_part"], dc_ref, rtol=1e-8,
                               atol=1e-9 * np.abs(dc_ref).max())
