"""Golden iterative_map run of BASELINE.json configs[1] (synthetic driving
sequence: 500 frames, 100k tracks, ~1M observations, 5% outliers) from the
vectorised oracle restatement (oracle/imap.py: mapping.py:569-624 with the
pinned BA restatement oracle/ba.py; both checked against sfmkit's own
iterative_map / ransac_triangulate outputs in tests/test_oracle_golden.py).
sfmkit itself needs hours for one round at this size (2.4-13 ms per track,
SURVEY.md section 6).

Inputs are exactly those of
tests/test_gpu_configs.py::test_config2_iterative_map_matches_oracle:
config_scene(2, seed=0), MappingConfig() defaults (stage 1 Huber 2 / 4 px,
stage 2 trivial / 2 px, lambda_c = lambda_a = 1, DLT), lambda_c edges between
consecutive frames, lambda_a priors on every non-fixed frame.

Stored (tests/golden/config2_imap.npz): status [T] int8, lm_track [L] int32,
inlier_mask packed bits [N], round statistics, final poses, a fixed sample
of landmark positions, and the per-BA LM reports.

    python tests/golden/make_config2_imap.py [out.npz]
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

MODELS = [(0, 500.0, 500.0, 320.0, 240.0, (0.0, 0.0))]


def inputs():
    from paper_2510_15271_b200.scenes import config_scene
    sc = config_scene(2, seed=0)
    ptr = np.searchsorted(sc.obs_point, np.arange(sc.n_points + 1)).astype(np.int64)
    F = sc.n_frames
    edges = np.stack([np.arange(F - 1), np.arange(1, F)], 1).astype(np.int32)
    priors = np.flatnonzero(sc.frame_fixed == 0).astype(np.int32)
    return sc, ptr, edges, priors


def main(out):
    from oracle import imap as OI
    t0 = time.time()
    sc, ptr, edges, priors = inputs()
    print(f"scene: {sc.n_frames} frames, {sc.n_points} tracks, {sc.n_obs} obs", flush=True)
    r = OI.iterative_map(sc.cam_q, sc.cam_t, np.zeros(sc.n_frames, np.int64), sc.frame_fixed,
                         MODELS, ptr, sc.obs_frame, sc.obs_uv, edges, priors,
                         log=lambda s: print(f"{s} ({time.time() - t0:.0f} s)", flush=True))
    lm = r["lm_track"]
    rng = np.random.default_rng(7)
    sample = np.sort(rng.choice(len(lm), size=min(2000, len(lm)), replace=False))
    rs = r["round_stats"]
    np.savez_compressed(
        out, status=r["status"].astype(np.int8), lm_track=lm.astype(np.int32),
        mask_bits=np.packbits(r["inlier_mask"]), n_obs=len(r["inlier_mask"]),
        round_stats=json.dumps(rs), cam_q=r["cam_q"], cam_t=r["cam_t"],
        lm_sample=sample, lm_sample_X=r["points"][lm[sample]],
        reports=json.dumps(r["reports"]))
    print(f"done in {time.time() - t0:.0f} s: {rs} -> {out}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "config2_imap.npz"))
