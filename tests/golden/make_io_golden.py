"""Golden outputs of sfmkit's writers (io.py:271-337 write_colmap_sparse,
:508-537 write_map) on the final map of the reference iterative_map fixture
(tests/golden/iterative_map.npz): the three COLMAP text files and the
map.bin bytes, for tests/test_cpu_host.py / tests/test_gpu_parity.py to
compare this package's writers (paper_2510_15271_b200/io.py) against.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py
"""
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import sfmkit.cameras as RC  # noqa: E402
import sfmkit.io as RIO  # noqa: E402
import sfmkit.keyframes as RK  # noqa: E402
import sfmkit.mapping as RM  # noqa: E402
import sfmkit.se3 as RS  # noqa: E402


def reference_map(d):
    ptr, lm_track = d["track_ptr"], d["ref_lm_track"]
    masks = np.split(d["ref_lm_mask"].astype(bool), np.cumsum([ptr[t + 1] - ptr[t] for t in lm_track])[:-1])
    cams = {0: RC.CameraModel("pinhole", 500.0, 500.0, 320.0, 240.0, 640, 480),
            1: RC.CameraModel("pinhole_radial", 480.0, 490.0, 321.5, 239.5, 640, 480, (-0.05, 0.01))}
    F = len(d["cam_q"])
    kfs = {f: RK.Keyframe(f, 0.1 * f, f % 2, RS.Pose(d["ref_cam_q"][f], d["ref_cam_t"][f]),
                          image_path=f"img/{f:04d}.jpg" if f % 3 else "") for f in range(F)}
    lms = []
    for i, t in enumerate(lm_track):
        obs = [RM.Observation(int(d["obs_frame"][o]), int(o), d["obs_uv"][o]) for o in range(ptr[t], ptr[t + 1])]
        lms.append(RM.Landmark(d["ref_lm_X"][i], RM.Track(obs, status="triangulated"), masks[i]))
    return RM.SparseMap(kfs, cams, lms, None, {1: "prior"}, {0})


def main(out=os.path.join(HERE, "io_writers.npz")):
    d = np.load(os.path.join(HERE, "iterative_map.npz"))
    m = reference_map(d)
    with tempfile.TemporaryDirectory() as td:
        RIO.write_colmap_sparse(m, td)
        files = {n: open(os.path.join(td, n), "rb").read() for n in ("cameras.txt", "images.txt", "points3D.txt")}
        RIO.write_map(m, os.path.join(td, "map.bin"))
        mb = open(os.path.join(td, "map.bin"), "rb").read()
    np.savez_compressed(out, cameras_txt=np.frombuffer(files["cameras.txt"], np.uint8),
                        images_txt=np.frombuffer(files["images.txt"], np.uint8),
                        points3d_txt=np.frombuffer(files["points3D.txt"], np.uint8),
                        map_bin=np.frombuffer(mb, np.uint8))
    print("wrote", out, {k: len(v) for k, v in files.items()}, len(mb))


if __name__ == "__main__":
    main()
