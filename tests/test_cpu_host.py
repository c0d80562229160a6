"""Host-side checks that need no GPU: the C-ABI library loads and exports
every symbol include/sfm_b200.h declares, the flattening contract, the
drop-in's pre-call errors, and the point-shard partitioner."""

import os
import re

import numpy as np
import pytest

from paper_2510_15271_b200 import _native as nat

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(REPO, "include", "sfm_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|void|const char\*)\s+(sfm_\w+)\(", src, re.M)))


def test_header_and_binding_agree():
    assert sorted(nat.EXPORTED_SYMBOLS) == header_functions()


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("libsfm_b200.so not built (run __graft_entry__.build())")
    lib = nat.load_library()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.sfm_abi_version() == nat.ABI_VERSION


def test_ctypes_struct_layout_matches_header(tmp_path):
    """sizeof / offsetof of every C-ABI struct, as gcc sees include/sfm_b200.h,
    equals the ctypes mirror in _native.py."""
    import ctypes
    import subprocess
    structs = {"sfm_camera_model": nat.CameraModelC, "sfm_ba_problem": nat.BAProblemC,
               "sfm_ba_options": nat.BAOptionsC, "sfm_ba_report": nat.BAReportC,
               "sfm_tracks": nat.TracksC, "sfm_map_problem": nat.MapProblemC,
               "sfm_map_options": nat.MapOptionsC, "sfm_round_stat": nat.RoundStatC,
               "sfm_gba_problem": nat.GbaProblemC}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "sfm_b200.h"', "int main(void){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(ln.rsplit(" ", 1) for ln in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_flatten_matches_golden_order(golden):
    """flatten_ba on the object model reproduces the fixture arrays, whose
    order the oracle tests pin to the reference residual order."""
    from paper_2510_15271_b200 import (CameraModel, Keyframe, Landmark, MappingConfig,
                                       Observation, Pose, SparseMap, Track, flatten_ba)
    d = golden("ba_cauchy_pose_terms")
    cam = CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
    F = len(d["cam_q"])
    kfs = {f: Keyframe(f, float(f), 0, Pose(d["cam_q"][f], d["cam_t"][f])) for f in range(F)}
    smap = SparseMap(kfs, {0: cam}, fixed_frames={int(f) for f in np.flatnonzero(d["frame_fixed"])})
    ptr = np.searchsorted(d["obs_point"], np.arange(len(d["points"]) + 1))
    for p in range(len(d["points"])):
        obs = [Observation(int(d["obs_frame"][o]), 0, d["obs_uv"][o]) for o in range(ptr[p], ptr[p + 1])]
        smap.landmarks.append(Landmark(d["points"][p], Track(obs, "triangulated"),
                                       np.ones(len(obs), bool)))
    from paper_2510_15271_b200.solver import RobustLoss
    from paper_2510_15271_b200.mapping import StageConfig
    cfg = MappingConfig(stage1=StageConfig(4.0, RobustLoss("cauchy", 1.5)), lambda_c=2.0,
                        lambda_a=0.5)
    a, frames, lms, loss = flatten_ba(smap, cfg, 1)
    np.testing.assert_array_equal(a.obs_frame, d["obs_frame"])
    np.testing.assert_array_equal(a.obs_point, d["obs_point"])
    np.testing.assert_array_equal(a.obs_uv, d["obs_uv"])
    np.testing.assert_array_equal(a.edge_ab, d["edge_ab"])
    np.testing.assert_array_equal(a.prior_frame, d["prior_frame"])
    assert loss.kind == "cauchy"


def test_flatten_skips_outlier_and_untriangulated():
    from paper_2510_15271_b200 import (CameraModel, Keyframe, Landmark, MappingConfig,
                                       Observation, Pose, SparseMap, Track, flatten_ba)
    cam = CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
    kfs = {f: Keyframe(f, float(f), 0, Pose()) for f in (3, 1, 2)}
    smap = SparseMap(kfs, {0: cam}, fixed_frames={1})
    obs = [Observation(f, 0, (10.0 * f, 5.0)) for f in (1, 2, 3)]
    smap.landmarks.append(Landmark([0, 0, 5], Track(list(obs), "triangulated"), [True, False, True]))
    smap.landmarks.append(Landmark([0, 0, 6], Track(list(obs), "pending"), [True, True, True]))
    smap.landmarks.append(Landmark([0, 0, 7], Track(list(obs), "triangulated"), [True, True, True]))
    a, frames, lms, _ = flatten_ba(smap, MappingConfig(), 1)
    assert frames == [1, 2, 3] and lms == [0, 2]
    np.testing.assert_array_equal(a.obs_point, [0, 0, 1, 1, 1])
    np.testing.assert_array_equal(a.obs_frame, [0, 2, 0, 1, 2])
    np.testing.assert_array_equal(a.frame_fixed, [1, 0, 0])
    np.testing.assert_array_equal(a.edge_ab, [[0, 1], [1, 2]])
    np.testing.assert_array_equal(a.prior_frame, [1, 2])


def test_no_gauge_raised_before_device_call():
    from paper_2510_15271_b200 import (CameraModel, Keyframe, MappingConfig, NoGauge, Pose,
                                       SparseMap, bundle_adjust)
    cam = CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
    smap = SparseMap({0: Keyframe(0, 0.0, 0, Pose())}, {0: cam})
    with pytest.raises(NoGauge):
        bundle_adjust(smap, MappingConfig(lambda_a=0.0, lambda_c=0.0), stage=2)


def test_single_slot_flatten_rejects_two_slot_problems():
    """flatten_ba is the single-slot (global-shutter, non-rig) layout;
    bundle_adjust routes rolling-shutter / rig problems to sfm_gba_solve."""
    from paper_2510_15271_b200 import (CameraModel, Keyframe, MappingConfig, Pose, SparseMap,
                                       flatten_ba)
    cam = CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
    kfs = {0: Keyframe(0, 0.0, 0, Pose(), shutter="rolling", exposure=0.03),
           1: Keyframe(1, 0.1, 0, Pose())}
    smap = SparseMap(kfs, {0: cam}, fixed_frames={0})
    with pytest.raises(NotImplementedError):
        flatten_ba(smap, MappingConfig(), 1)
    with pytest.raises(NotImplementedError):
        flatten_ba(SparseMap({0: Keyframe(0, 0.0, 0, Pose())}, {0: cam}, fixed_frames={0}),
                   MappingConfig(), 1, mode="rig_extrinsic")


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_ranges_balanced_and_contiguous(world):
    from paper_2510_15271_b200.mapping import shard_ranges
    rng = np.random.default_rng(world)
    k = rng.integers(2, 12, 5000)
    obs_point = np.repeat(np.arange(5000), k)
    rs = shard_ranges(obs_point, 5000, world)
    assert rs[0][0] == 0 and rs[-1][1] == 5000
    for (a, b), (c, _) in zip(rs, rs[1:]):
        assert b == c and a <= b
    counts = [int(k[a:b].sum()) for a, b in rs]
    assert max(counts) - min(counts) <= 2 * k.max()


def test_scene_generator_layout():
    from paper_2510_15271_b200.scenes import make_scene
    sc = make_scene(40, 3000, 15000, shape="venice", seed=2, outlier_frac=0.05)
    assert np.all(np.diff(sc.obs_point) >= 0)
    # frames strictly increasing inside each track (build_tracks order)
    same = sc.obs_point[1:] == sc.obs_point[:-1]
    assert np.all(np.diff(sc.obs_frame)[same] > 0)
    assert np.bincount(sc.obs_point).min() >= 2
    assert 0 < sc.outlier.mean() < 0.1


# --- build_tracks (host-native, mapping.py:113-161): runs without a GPU -----

def test_build_tracks_matches_reference_fixture(golden):
    """sfm_build_tracks against sfmkit's build_tracks on a random match graph
    with conflicting joins (tests/golden/make_golden.py): bit-exact CSR."""
    from paper_2510_15271_b200.mapping import build_tracks_arrays
    d = golden("build_tracks")
    tp, of, fi = build_tracks_arrays(d["pair_frames"], d["pair_ptr"], d["match_index"])
    np.testing.assert_array_equal(tp, d["ref_track_ptr"])
    np.testing.assert_array_equal(of, d["ref_obs_frame"])
    np.testing.assert_array_equal(fi, d["ref_obs_feature"])


class _KP:
    def __init__(self, x, y):
        self.x, self.y = x, y


class _Feats:
    def __init__(self, n):
        self.keypoints = [_KP(10.0 * i, 5.0 * i) for i in range(n)]


class _M:
    def __init__(self, a, b):
        self.index_a, self.index_b = a, b


def test_build_tracks_transitive_chain():
    from paper_2510_15271_b200.mapping import PENDING, build_tracks
    feats = {f: _Feats(4) for f in range(3)}
    tracks = build_tracks({(0, 1): [_M(0, 0)], (1, 2): [_M(0, 0)]}, feats)
    assert len(tracks) == 1
    assert [(o.frame_id, o.feature_index) for o in tracks[0].observations] == [(0, 0), (1, 0), (2, 0)]
    assert tracks[0].status == PENDING
    assert tracks[0].observations[1].pixel.tolist() == [0.0, 0.0]


def test_build_tracks_conflict_split():
    from paper_2510_15271_b200.mapping import build_tracks
    feats = {f: _Feats(6) for f in range(3)}
    tracks = build_tracks({(0, 1): [_M(0, 0)], (0, 2): [_M(1, 5)], (1, 2): [_M(0, 5)]}, feats)
    assert len(tracks) == 2
    nodes = sorted((o.frame_id, o.feature_index) for t in tracks for o in t.observations)
    assert nodes == [(0, 0), (0, 1), (1, 0), (2, 5)]
    for t in tracks:
        frames = [o.frame_id for o in t.observations]
        assert len(frames) == len(set(frames))


def test_build_tracks_matches_union_find():
    from paper_2510_15271_b200.mapping import build_tracks
    rng = np.random.default_rng(42)
    n_frames, n_feat = 6, 12
    feats = {f: _Feats(n_feat) for f in range(n_frames)}
    pairs = {(f, f + 1): [_M(int(k), int(k)) for k in sorted(rng.choice(n_feat, 7, replace=False))]
             for f in range(n_frames - 1)}
    parent = {}

    def find(x):
        while parent.setdefault(x, x) != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x
    for (fa, fb), ms in pairs.items():
        for m in ms:
            parent[find((fa, m.index_a))] = find((fb, m.index_b))
    comps = {}
    for node in list(parent):
        comps.setdefault(find(node), set()).add(node)
    expected = sorted(sorted(c) for c in comps.values() if len(c) >= 2)
    got = sorted(sorted((o.frame_id, o.feature_index) for o in t.observations)
                 for t in build_tracks(pairs, feats))
    assert got == expected


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not mounted (GPU box)")
def test_dropin_map_writes_reference_map_bin(tmp_path, golden):
    """The drop-in's object model is what sfmkit's `map` stage serialises:
    sfmkit.io.write_map on this package's SparseMap (built from the
    reference iterative_map fixture) produces the same bytes as on the
    equivalent sfmkit SparseMap, and read_map round-trips it (SURVEY.md
    §8(f) row 4: map.bin compatibility)."""
    import sys
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    sys.dont_write_bytecode = True
    import sfmkit.cameras as RC
    import sfmkit.io as RIO
    import sfmkit.keyframes as RK
    import sfmkit.mapping as RM
    import sfmkit.se3 as RS
    from paper_2510_15271_b200 import (CameraModel, Keyframe, Landmark, Observation, Pose,
                                       SparseMap, Track)
    d = golden("iterative_map")
    ptr, lm_track = d["track_ptr"], d["ref_lm_track"]
    masks = np.split(d["ref_lm_mask"].astype(bool),
                     np.cumsum([ptr[t + 1] - ptr[t] for t in lm_track])[:-1])

    def build(Cam, Kf, Ps, Obs, Tr, Lm, Sm):
        cam = Cam("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480)
        kfs = {f: Kf(f, float(f), 0, Ps(d["ref_cam_q"][f], d["ref_cam_t"][f]))
               for f in range(len(d["cam_q"]))}
        lms = []
        for i, t in enumerate(lm_track):
            obs = [Obs(int(d["obs_frame"][o]), 0, d["obs_uv"][o]) for o in range(ptr[t], ptr[t + 1])]
            lms.append(Lm(d["ref_lm_X"][i], Tr(obs, status="triangulated"), masks[i]))
        return Sm(kfs, {0: cam}, lms, None, {}, {0})

    ours = build(CameraModel, Keyframe, Pose, Observation, Track, Landmark, SparseMap)
    ref = build(RC.CameraModel, RK.Keyframe, RS.Pose, RM.Observation, RM.Track, RM.Landmark,
                RM.SparseMap)
    RIO.write_map(ours, tmp_path / "ours.bin")
    RIO.write_map(ref, tmp_path / "ref.bin")
    assert (tmp_path / "ours.bin").read_bytes() == (tmp_path / "ref.bin").read_bytes()
    back = RIO.read_map(tmp_path / "ours.bin")
    assert len(back.landmarks) == len(ours.landmarks)
    np.testing.assert_array_equal(np.array([lm.position for lm in back.landmarks]), d["ref_lm_X"])


def _io_map(golden):
    """The map of tests/golden/make_io_golden.py in this package's objects."""
    from paper_2510_15271_b200 import (CameraModel, Keyframe, Landmark, Observation, Pose,
                                       SparseMap, Track)
    d = golden("iterative_map")
    ptr, lm_track = d["track_ptr"], d["ref_lm_track"]
    masks = np.split(d["ref_lm_mask"].astype(bool),
                     np.cumsum([ptr[t + 1] - ptr[t] for t in lm_track])[:-1])
    cams = {0: CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480),
            1: CameraModel("pinhole_radial", 480.0, 490.0, 321.5, 239.5, 640, 480, (-0.05, 0.01))}
    F = len(d["cam_q"])
    kfs = {f: Keyframe(f, 0.1 * f, f % 2, Pose(d["ref_cam_q"][f], d["ref_cam_t"][f]),
                       image_path=f"img/{f:04d}.jpg" if f % 3 else "") for f in range(F)}
    lms = []
    for i, t in enumerate(lm_track):
        obs = [Observation(int(d["obs_frame"][o]), int(o), d["obs_uv"][o]) for o in range(ptr[t], ptr[t + 1])]
        lms.append(Landmark(d["ref_lm_X"][i], Track(obs, status="triangulated"), masks[i]))
    return SparseMap(kfs, cams, lms, None, {1: "prior"}, {0})


def test_map_bin_writer_matches_reference_bytes(tmp_path, golden):
    """paper_2510_15271_b200.io.write_map: the same bytes as sfmkit's
    write_map (io.py:508-537, CRC32 container io.py:348-361) on the same map
    (tests/golden/io_writers.npz from tests/golden/make_io_golden.py), and
    read_map round-trips it."""
    from paper_2510_15271_b200 import io as SIO
    g = golden("io_writers")
    m = _io_map(golden)
    SIO.write_map(m, tmp_path / "map.bin")
    assert (tmp_path / "map.bin").read_bytes() == g["map_bin"].tobytes()
    back = SIO.read_map(tmp_path / "map.bin")
    assert SIO.map_bytes(back) == g["map_bin"].tobytes()
    bad = bytearray(g["map_bin"].tobytes())
    bad[40] ^= 1
    (tmp_path / "bad.bin").write_bytes(bytes(bad))
    with pytest.raises(SIO.ChecksumMismatch):
        SIO.read_map(tmp_path / "bad.bin")
