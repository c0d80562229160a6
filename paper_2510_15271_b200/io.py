"""Output writers on either side of the mapping path:
the checksummed `map.bin` container that `sfmkit map` writes
(io.py:348-361 container, :508-537 sparse map) and the COLMAP sparse text
triplet (io.py:271-337), byte-compatible with the reference's files.

The map is this package's object model (mapping.SparseMap, the same schema
as sfmkit's); the per-observation reprojection errors of the COLMAP
points3D ERROR column come from the device (sfm_reprojection_errors, the
kernel behind reprojection_error / remove_outliers).
"""

from __future__ import annotations

import json
import os
import struct
import zlib

import numpy as np

from .cameras import EQUIDISTANT_FISHEYE, PINHOLE, PINHOLE_RADIAL
from .mapping import TRIANGULATED, Landmark, Observation, SparseMap, Track

MAP_MAGIC = b"SFMMAP\0\0"     # io.py:346
FORMAT_VERSION = 1            # io.py:30


class ChecksumMismatch(ValueError):
    """Container whose CRC32 does not match (sfmkit.errors.ChecksumMismatch)."""


try:  # the reference's own class when sfmkit is importable (same except clauses work)
    from sfmkit.errors import ChecksumMismatch  # type: ignore  # noqa: F811
except ImportError:
    pass


# --- container: magic(8) version(u32) count(u32) [name(16) len(u64)]* payload crc32(u32)

def _pack_container(magic: bytes, sections) -> bytes:
    head = bytearray(magic)
    head += struct.pack("<II", FORMAT_VERSION, len(sections))
    blobs = bytearray()
    for name, blob in sections:
        key = name.encode("ascii")
        if len(key) > 16:
            raise ValueError(f"section name too long: {name}")
        head += key + b"\0" * (16 - len(key)) + struct.pack("<Q", len(blob))
        blobs += blob
    body = bytes(head + blobs)
    return body + struct.pack("<I", zlib.crc32(body))


def _unpack_container(data: bytes, magic: bytes) -> dict:
    if len(data) < 20:
        raise ChecksumMismatch("file too short")
    body = data[:-4]
    if zlib.crc32(body) != struct.unpack("<I", data[-4:])[0]:
        raise ChecksumMismatch("crc32 mismatch")
    if body[:8] != magic:
        raise ValueError("wrong magic")
    version, count = struct.unpack("<II", body[8:16])
    if version != FORMAT_VERSION:
        raise ValueError(f"unsupported format version {version}")
    at = 16
    entries = []
    for _ in range(count):
        name = body[at:at + 16].rstrip(b"\0").decode("ascii")
        (n,) = struct.unpack("<Q", body[at + 16:at + 24])
        entries.append((name, n))
        at += 24
    out = {}
    for name, n in entries:
        out[name] = body[at:at + n]
        at += n
    return out


def _json(obj) -> bytes:
    # sorted keys, no whitespace (io.py:392-393): the bytes are the format
    return json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()


def _pose(p):
    return {"quat": [float(v) for v in p.quat], "t": [float(v) for v in p.t]}


def _camera(cid, cam):
    return {"id": int(cid), "kind": cam.kind, "fx": cam.fx, "fy": cam.fy, "cx": cam.cx,
            "cy": cam.cy, "width": cam.width, "height": cam.height,
            "distortion": list(cam.distortion)}


def map_bytes(sparse_map: SparseMap) -> bytes:
    """The map.bin bytes of `sparse_map` (write_map, io.py:508-537)."""
    kfs = sparse_map.keyframes
    doc = {
        "cameras": [_camera(c, sparse_map.cameras[c]) for c in sorted(sparse_map.cameras)],
        "keyframes": [{"frame_id": int(kfs[f].frame_id), "timestamp": float(kfs[f].timestamp),
                       "camera_id": int(kfs[f].camera_id), "cam_from_world": _pose(kfs[f].cam_from_world),
                       "image": kfs[f].image_path, "shutter": kfs[f].shutter,
                       "exposure": float(kfs[f].exposure)} for f in sorted(kfs)],
        "landmarks": [{"position": [float(v) for v in lm.position], "status": lm.track.status,
                       "observations": [{"frame_id": int(o.frame_id),
                                         "feature_index": int(o.feature_index),
                                         "pixel": [float(o.pixel[0]), float(o.pixel[1])]}
                                        for o in lm.track.observations],
                       "inliers": [bool(b) for b in lm.inlier_mask]}
                      for lm in sparse_map.landmarks],
        "provenance": {str(int(f)): sparse_map.provenance[f] for f in sorted(sparse_map.provenance)},
        "fixed_frames": sorted(int(f) for f in sparse_map.fixed_frames),
        "rig": None,
    }
    rig = sparse_map.rig
    if rig is not None:
        doc["rig"] = {"camera_ids": [int(c) for c in rig.camera_ids],
                      "cam_from_rig": {str(int(c)): _pose(rig.extrinsic(c)) for c in rig.camera_ids}}
    return _pack_container(MAP_MAGIC, [("map", _json(doc))])


def write_map(sparse_map: SparseMap, path) -> None:
    """io.py:508-537: the map as one JSON section in the CRC32 container."""
    with open(path, "wb") as f:
        f.write(map_bytes(sparse_map))


def read_map(path) -> SparseMap:
    """io.py:540-565 into this package's object model."""
    from .cameras import CameraModel, RigCalibration
    from .keyframes import Keyframe
    from .se3 import Pose
    with open(path, "rb") as f:
        doc = json.loads(_unpack_container(f.read(), MAP_MAGIC)["map"])
    cams = {int(c["id"]): CameraModel(c["kind"], float(c["fx"]), float(c["fy"]), float(c["cx"]),
                                      float(c["cy"]), int(c["width"]), int(c["height"]),
                                      tuple(c.get("distortion", ())))
            for c in doc["cameras"]}
    kfs = {}
    for k in doc["keyframes"]:
        p = k["cam_from_world"]
        kfs[k["frame_id"]] = Keyframe(k["frame_id"], k["timestamp"], k["camera_id"],
                                      Pose(np.asarray(p["quat"], float), np.asarray(p["t"], float)),
                                      image_path=k["image"], shutter=k["shutter"],
                                      exposure=k["exposure"])
    rig = None
    if doc["rig"] is not None:
        ids = tuple(int(c) for c in doc["rig"]["camera_ids"])
        rig = RigCalibration(ids, {c: Pose(np.asarray(doc["rig"]["cam_from_rig"][str(c)]["quat"], float),
                                           np.asarray(doc["rig"]["cam_from_rig"][str(c)]["t"], float))
                                   for c in ids})
    lms = []
    for item in doc["landmarks"]:
        obs = [Observation(o["frame_id"], o["feature_index"], o["pixel"]) for o in item["observations"]]
        lms.append(Landmark(np.asarray(item["position"]), Track(obs, status=item["status"]),
                            np.asarray(item["inliers"], dtype=bool)))
    return SparseMap(kfs, cams, lms, rig, {int(f): v for f, v in doc["provenance"].items()},
                     set(doc["fixed_frames"]))


# --- COLMAP sparse text (io.py:247-337) --------------------------------------

COLMAP_MODEL = {PINHOLE: "PINHOLE", PINHOLE_RADIAL: "OPENCV", EQUIDISTANT_FISHEYE: "OPENCV_FISHEYE"}


def _g(v) -> str:
    return f"{v:.9g}"


def _colmap_params(cam):
    p = [cam.fx, cam.fy, cam.cx, cam.cy]
    if cam.kind == PINHOLE_RADIAL:
        p += [cam.distortion[0], cam.distortion[1], 0.0, 0.0]
    elif cam.kind == EQUIDISTANT_FISHEYE:
        p += [0.0, 0.0, 0.0, 0.0]
    return p


def write_colmap_sparse(sparse_map: SparseMap, out_dir, ctx=None) -> None:
    """cameras.txt / images.txt / points3D.txt with 1-based point ids in map
    order over the TRIANGULATED landmarks, each image's 2-D points in
    landmark order, and per point the mean reprojection error of its inlier
    observations (computed on the device)."""
    from .mapping import _reproj_errors
    for cam in sparse_map.cameras.values():
        if cam.kind not in COLMAP_MODEL:
            raise ValueError(f"unsupported camera kind {cam.kind!r}")
    os.makedirs(out_dir, exist_ok=True)
    tri = [li for li, lm in enumerate(sparse_map.landmarks) if lm.track.status == TRIANGULATED]
    pid = {li: k + 1 for k, li in enumerate(tri)}
    per_image = {f: [] for f in sparse_map.keyframes}      # (x, y, point id, landmark)
    inl = {}
    for li in tri:
        lm = sparse_map.landmarks[li]
        inl[li] = lm.inlier_observations()
        for o in inl[li]:
            per_image[o.frame_id].append((o.pixel[0], o.pixel[1], pid[li], li))
    refs = {li: [] for li in tri}                           # (image id, point2D index)
    for f in sorted(per_image):
        for k, (_, _, _, li) in enumerate(per_image[f]):
            refs[li].append((f, k))
    poses = {f: kf.cam_from_world for f, kf in sparse_map.keyframes.items()}
    cams = {f: sparse_map.camera_of(f) for f in sparse_map.keyframes}
    errs = {}
    lists = [inl[li] for li in tri if inl[li]]
    if lists:
        pos = np.array([sparse_map.landmarks[li].position for li in tri if inl[li]])
        e, _ = _reproj_errors(lists, pos, poses, cams, ctx)
        at = 0
        for li in (li for li in tri if inl[li]):
            n = len(inl[li])
            errs[li] = float(np.mean(list(e[at:at + n])))
            at += n
    with open(os.path.join(out_dir, "cameras.txt"), "w") as f:
        f.write("# Camera list with one line of data per camera:\n"
                "#   CAMERA_ID, MODEL, WIDTH, HEIGHT, PARAMS[]\n")
        for cid in sorted(sparse_map.cameras):
            cam = sparse_map.cameras[cid]
            f.write(f"{cid} {COLMAP_MODEL[cam.kind]} {cam.width} {cam.height} "
                    + " ".join(_g(v) for v in _colmap_params(cam)) + "\n")
    with open(os.path.join(out_dir, "images.txt"), "w") as f:
        f.write("# Image list with two lines of data per image:\n"
                "#   IMAGE_ID, QW, QX, QY, QZ, TX, TY, TZ, CAMERA_ID, NAME\n"
                "#   POINTS2D[] as (X, Y, POINT3D_ID)\n")
        for fid in sorted(sparse_map.keyframes):
            kf = sparse_map.keyframes[fid]
            q, t = kf.cam_from_world.quat, kf.cam_from_world.t
            name = kf.image_path or f"frame{fid:06d}.png"
            f.write(" ".join([str(fid)] + [_g(v) for v in (q[0], q[1], q[2], q[3], t[0], t[1], t[2])]
                             + [str(kf.camera_id), name]) + "\n")
            f.write(" ".join(f"{_g(x)} {_g(y)} {p}" for x, y, p, _ in per_image[fid]) + "\n")
    with open(os.path.join(out_dir, "points3D.txt"), "w") as f:
        f.write("# 3D point list with one line of data per point:\n"
                "#   POINT3D_ID, X, Y, Z, R, G, B, ERROR, TRACK[] as (IMAGE_ID, POINT2D_IDX)\n")
        for li in tri:
            X = sparse_map.landmarks[li].position
            track = " ".join(f"{img} {k}" for img, k in refs[li])
            f.write(f"{pid[li]} {_g(X[0])} {_g(X[1])} {_g(X[2])} 128 128 128 "
                    f"{_g(errs.get(li, 0.0))} {track}\n")
