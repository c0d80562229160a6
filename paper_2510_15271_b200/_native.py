"""ctypes binding to libsfm_b200.so (include/sfm_b200.h).

The shared library is built in-tree (``__graft_entry__.build()`` or
``make -C paper_2510_15271_b200/csrc``).  There is no CPU fallback: if the
library is missing or no CUDA device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsfm_b200.so")

# ---- constants (mirror include/sfm_b200.h) ---------------------------------
ABI_VERSION = 7
SFM_OK = 0
SFM_E_INVALID = -1
SFM_E_NON_POSITIVE_DEPTH = -2
SFM_E_OUT_OF_MODEL_DOMAIN = -3
SFM_E_SOLVER_DIVERGED = -4
SFM_E_UNDISTORT_DIVERGED = -5
SFM_E_NO_GAUGE = -6
SFM_E_CUDA = -10
SFM_E_NCCL = -11
SFM_E_OOM = -12

TRI_OK = 0
TRI_INSUFFICIENT_PARALLAX = 1
TRI_CHEIRALITY = 2
TRI_PARALLEL_RAYS = 3
TRI_TOO_FEW_OBS = 4
TRI_CAMERA_ERROR = 5
TRI_FAILED = 6
TRI_SKIPPED = 7
TRI_CAMERA_DOMAIN = 8

CAM_KINDS = {"pinhole": 0, "pinhole_radial": 1, "equidistant_fisheye": 2}
LOSS_KINDS = {"trivial": 0, "huber": 1, "cauchy": 2}
LINSOLVE = {"auto": 0, "dense": 1, "pcg": 2}
TERMINATIONS = ("max_iterations", "gradient_tolerance", "no_decrease",
                "parameter_tolerance", "cost_zero", "all_fixed")
TRI_METHODS = {"dlt": 0, "midpoint": 1}


def tri_method(method: str) -> int:
    """ransac_triangulate's `method` (mapping.py:270-278): "dlt" is the DLT,
    every other value the midpoint method."""
    return 0 if method == "dlt" else 1

EXPORTED_SYMBOLS = (
    "sfm_abi_version", "sfm_nccl_unique_id", "sfm_ctx_create", "sfm_ctx_create_multi",
    "sfm_ctx_devices", "sfm_device_count", "sfm_ctx_destroy",
    "sfm_last_error", "sfm_ctx_stream", "sfm_set_profiling", "sfm_prof_count", "sfm_prof_get",
    "sfm_prof_reset", "sfm_ba_solve", "sfm_ba_setup", "sfm_ba_iterate",
    "sfm_ba_download", "sfm_ba_restart", "sfm_ba_eval", "sfm_ransac_triangulate", "sfm_triangulate",
    "sfm_gate", "sfm_reprojection_errors", "sfm_iterative_map", "sfm_ba_solve_emulated",
    "sfm_build_tracks", "sfm_gba_solve", "sfm_shard_points", "sfm_pcg_rank_rows",
)

TRACK_PENDING, TRACK_TRIANGULATED, TRACK_FAILED = 0, 1, 2
RES_GLOBAL, RES_ROLLING, RES_RIG = 0, 1, 2

_p = ctypes.c_void_p


class CameraModelC(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("width", ctypes.c_int32),
                ("height", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("k1", ctypes.c_double), ("k2", ctypes.c_double)]


class BAProblemC(ctypes.Structure):
    _fields_ = [("n_frames", ctypes.c_int32), ("n_models", ctypes.c_int32),
                ("cam_q", _p), ("cam_t", _p), ("frame_model", _p),
                ("frame_fixed", _p), ("models", _p),
                ("n_points", ctypes.c_int64), ("points", _p),
                ("n_obs", ctypes.c_int64), ("obs_frame", _p), ("obs_point", _p),
                ("obs_uv", _p),
                ("n_edges", ctypes.c_int32), ("n_priors", ctypes.c_int32),
                ("edge_ab", _p), ("prior_frame", _p),
                ("edge_weight", ctypes.c_double), ("prior_weight", ctypes.c_double),
                ("obs_offset", ctypes.c_int64), ("n_params_global", ctypes.c_int64)]


class BAOptionsC(ctypes.Structure):
    _fields_ = [("loss_kind", ctypes.c_int32), ("max_iters", ctypes.c_int32),
                ("loss_param", ctypes.c_double), ("grad_tol", ctypes.c_double),
                ("param_tol", ctypes.c_double), ("initial_lambda", ctypes.c_double),
                ("max_lambda", ctypes.c_double), ("linear_solver", ctypes.c_int32),
                ("pcg_max_iters", ctypes.c_int32), ("pcg_rtol", ctypes.c_double),
                ("dense_max_dim", ctypes.c_int32), ("coarse_cluster", ctypes.c_int32),
                ("coarse_refresh", ctypes.c_int32), ("coarse_max_lambda", ctypes.c_double),
                ("coarse_drift", ctypes.c_double), ("pcg_partition", ctypes.c_int32),
                ("_pad0", ctypes.c_int32)]


class BAReportC(ctypes.Structure):
    _fields_ = [("initial_cost", ctypes.c_double), ("final_cost", ctypes.c_double),
                ("iterations", ctypes.c_int32), ("termination", ctypes.c_int32),
                ("n_trials", ctypes.c_int32), ("pcg_iterations", ctypes.c_int32),
                ("final_lambda", ctypes.c_double), ("device_ms", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64), ("n_blocks_S", ctypes.c_int64),
                ("pcg_stagnated", ctypes.c_int32), ("pcg_max_hit", ctypes.c_int32)]


class TracksC(ctypes.Structure):
    _fields_ = [("n_frames", ctypes.c_int32), ("n_models", ctypes.c_int32),
                ("cam_q", _p), ("cam_t", _p), ("frame_model", _p), ("models", _p),
                ("n_tracks", ctypes.c_int64), ("n_obs", ctypes.c_int64),
                ("track_ptr", _p), ("obs_frame", _p), ("obs_uv", _p), ("active", _p)]


class GbaProblemC(ctypes.Structure):
    _fields_ = [("n_blocks", ctypes.c_int32), ("n_models", ctypes.c_int32),
                ("block_q", _p), ("block_t", _p), ("block_fixed", _p), ("models", _p),
                ("n_points", ctypes.c_int64), ("points", _p), ("n_res", ctypes.c_int64),
                ("res_point", _p), ("res_model", _p), ("res_kind", _p), ("res_slot", _p),
                ("res_alpha", _p), ("res_uv", _p), ("n_edges", ctypes.c_int32),
                ("n_priors", ctypes.c_int32), ("edge_ab", _p), ("edge_weight", _p),
                ("prior_block", _p), ("prior_weight", _p)]


class MapProblemC(ctypes.Structure):
    _fields_ = [("n_frames", ctypes.c_int32), ("n_models", ctypes.c_int32),
                ("cam_q", _p), ("cam_t", _p), ("frame_model", _p), ("frame_fixed", _p),
                ("models", _p), ("n_tracks", ctypes.c_int64), ("n_obs", ctypes.c_int64),
                ("track_ptr", _p), ("obs_frame", _p), ("obs_uv", _p), ("track_status", _p),
                ("n_edges", ctypes.c_int32), ("n_priors", ctypes.c_int32),
                ("edge_ab", _p), ("prior_frame", _p),
                ("edge_weight", ctypes.c_double), ("prior_weight", ctypes.c_double)]


class MapOptionsC(ctypes.Structure):
    _fields_ = [("max_outer_iters", ctypes.c_int32), ("max_solver_iters", ctypes.c_int32),
                ("stage1_loss_kind", ctypes.c_int32), ("stage2_loss_kind", ctypes.c_int32),
                ("stage1_loss_param", ctypes.c_double), ("stage2_loss_param", ctypes.c_double),
                ("stage1_outlier_px", ctypes.c_double), ("stage2_outlier_px", ctypes.c_double),
                ("min_angle", ctypes.c_double), ("method", ctypes.c_int32),
                ("_pad", ctypes.c_int32), ("solver", BAOptionsC)]


class RoundStatC(ctypes.Structure):
    _fields_ = [("round", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("added", ctypes.c_int64), ("removed", ctypes.c_int64),
                ("landmarks", ctypes.c_int64)]


_lib = None
_lib_lock = threading.Lock()


class NativeLibraryMissing(RuntimeError):
    pass


def load_library(path: str = None):
    """Loads (once) and returns the ctypes handle; raises if absent."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        # SFM_B200_LIB: an alternative in-tree build (A/B experiments)
        path = path or os.environ.get("SFM_B200_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise NativeLibraryMissing(
                f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(no CPU fallback exists for this path)")
        lib = ctypes.CDLL(path)
        c_int, c_i32, c_i64, c_d = ctypes.c_int, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        P = ctypes.POINTER
        lib.sfm_abi_version.restype = c_int
        lib.sfm_nccl_unique_id.argtypes = [ctypes.c_char_p]
        lib.sfm_ctx_create.argtypes = [c_i32, c_i32, c_i32, ctypes.c_char_p, P(_p)]
        lib.sfm_ctx_destroy.argtypes = [_p]
        lib.sfm_ctx_destroy.restype = None
        lib.sfm_last_error.argtypes = [_p]
        lib.sfm_last_error.restype = ctypes.c_char_p
        lib.sfm_set_profiling.argtypes = [_p, c_i32]
        lib.sfm_prof_count.argtypes = [_p]
        lib.sfm_prof_get.argtypes = [_p, c_i32, P(ctypes.c_char_p), P(c_i64), P(c_d), P(c_d)]
        lib.sfm_prof_reset.argtypes = [_p]
        lib.sfm_ba_solve.argtypes = [_p, P(BAProblemC), P(BAOptionsC), _p, _p, _p, P(BAReportC)]
        lib.sfm_ba_setup.argtypes = [_p, P(BAProblemC), P(BAOptionsC)]
        lib.sfm_ba_iterate.argtypes = [_p, c_i32, P(BAReportC)]
        lib.sfm_ba_download.argtypes = [_p, _p, _p, _p]
        lib.sfm_ba_restart.argtypes = [_p]
        lib.sfm_ctx_stream.argtypes = [_p, P(_p)]
        lib.sfm_ctx_create_multi.argtypes = [c_i32, P(c_i32), P(_p)]
        lib.sfm_ctx_devices.argtypes = [_p, P(c_i32), P(c_i32)]
        lib.sfm_device_count.argtypes = [P(c_i32)]
        lib.sfm_ba_eval.argtypes = [_p, P(BAProblemC), c_i32, c_d, _p, _p, _p, _p]
        lib.sfm_ransac_triangulate.argtypes = [_p, P(TracksC), c_d, c_d, c_i32, _p, _p, _p]
        lib.sfm_triangulate.argtypes = [_p, P(TracksC), c_d, c_i32, _p, _p]
        lib.sfm_gate.argtypes = [_p, P(TracksC), _p, c_d, _p, _p, P(c_i64)]
        lib.sfm_reprojection_errors.argtypes = [_p, P(TracksC), _p, _p]
        lib.sfm_gba_solve.argtypes = [_p, P(GbaProblemC), P(BAOptionsC), _p, _p, _p, P(BAReportC)]
        lib.sfm_build_tracks.argtypes = [c_i64, _p, _p, _p, _p, _p, _p, P(c_i64), P(c_i64)]
        lib.sfm_shard_points.argtypes = [c_i64, _p, c_i64, c_i32, _p]
        lib.sfm_pcg_rank_rows.argtypes = [c_i32, _p, c_i32, _p]
        lib.sfm_ba_solve_emulated.argtypes = [_p, c_i32, _p, P(BAOptionsC), _p, _p, _p,
                                              P(BAReportC)]
        lib.sfm_iterative_map.argtypes = [_p, P(MapProblemC), P(MapOptionsC), _p, _p, _p, _p, _p,
                                          _p, P(c_i64), _p, P(c_i32)]
        for name in EXPORTED_SYMBOLS:
            if name not in ("sfm_ctx_destroy", "sfm_last_error"):
                getattr(lib, name).restype = c_int
        if lib.sfm_abi_version() != ABI_VERSION:
            raise NativeLibraryMissing("libsfm_b200.so ABI version mismatch")
        _lib = lib
        return lib


def ptr(a):
    """Raw data pointer of a C-contiguous numpy array (or None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the C-ABI must be C-contiguous"
    return a.ctypes.data


class Context:
    """One sfm_ctx: one CUDA device and stream, with an optional NCCL
    communicator (one process per GPU, `rank` of `world`) -- or, from
    Context.multi, every device of a single-process multi-GPU context."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: bytes = None, _handle=None, _devices=None):
        self.lib = load_library()
        self.device, self.rank, self.world = device, rank, world
        self.devices = list(_devices) if _devices else [device]
        if _handle is not None:
            self.handle = _handle
            return
        h = _p()
        rc = self.lib.sfm_ctx_create(device, rank, world, nccl_id, ctypes.byref(h))
        if rc != SFM_OK:
            raise RuntimeError(f"sfm_ctx_create failed (code {rc}); is a CUDA device visible?")
        self.handle = h

    @classmethod
    def multi(cls, devices) -> "Context":
        """Single-process multi-GPU context (sfm_ctx_create_multi): solves on
        it are point-sharded over `devices`, NCCL communicators created
        in-process; a repeated device id runs its ranks as shard emulation."""
        lib = load_library()
        devs = (ctypes.c_int32 * len(devices))(*[int(d) for d in devices])
        h = _p()
        rc = lib.sfm_ctx_create_multi(len(devices), devs, ctypes.byref(h))
        if rc != SFM_OK:
            raise RuntimeError(f"sfm_ctx_create_multi failed (code {rc})")
        return cls(int(devices[0]), 0, 1, _handle=h, _devices=devices)

    def topology(self):
        """(devices driven by this context, NCCL in use)."""
        n, nccl = ctypes.c_int32(), ctypes.c_int32()
        self.check(self.lib.sfm_ctx_devices(self.handle, ctypes.byref(n), ctypes.byref(nccl)))
        return n.value, bool(nccl.value)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.sfm_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> str:
        return self.lib.sfm_last_error(self.handle).decode(errors="replace")

    def check(self, rc: int):
        if rc != SFM_OK:
            from .errors import raise_for_code
            raise_for_code(rc, self.last_error())

    # profiling ----------------------------------------------------------
    def stream_handle(self) -> int:
        """cudaStream_t of this context (sfm_ctx_stream) as an integer."""
        out = _p()
        self.check(self.lib.sfm_ctx_stream(self.handle, ctypes.byref(out)))
        return int(out.value or 0)

    def set_profiling(self, on: bool):
        self.check(self.lib.sfm_set_profiling(self.handle, 1 if on else 0))

    def profile(self) -> dict:
        out = {}
        n = self.lib.sfm_prof_count(self.handle)
        for i in range(n):
            name = ctypes.c_char_p()
            launches = ctypes.c_int64()
            ms = ctypes.c_double()
            nbytes = ctypes.c_double()
            self.check(self.lib.sfm_prof_get(self.handle, i, ctypes.byref(name),
                                             ctypes.byref(launches), ctypes.byref(ms),
                                             ctypes.byref(nbytes)))
            out[name.value.decode()] = {"launches": launches.value, "ms": ms.value,
                                        "bytes": nbytes.value}
        return out

    def reset_profile(self):
        self.check(self.lib.sfm_prof_reset(self.handle))


def shard_points(obs_point, n_points: int, world: int) -> np.ndarray:
    """sfm_shard_points: point boundaries [world+1] of the observation-balanced
    point shards (host-only, no GPU)."""
    op = np.ascontiguousarray(obs_point, dtype=np.int32)
    out = np.empty(world + 1, np.int64)
    rc = load_library().sfm_shard_points(len(op), ptr(op), int(n_points), int(world), ptr(out))
    if rc != SFM_OK:
        raise ValueError(f"sfm_shard_points failed ({rc})")
    return out


def pcg_rank_rows(row_ptr, world: int) -> np.ndarray:
    """sfm_pcg_rank_rows: block-row boundaries [world+1] of the row-partitioned
    PCG over a BSR row pointer (host-only, no GPU)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    out = np.empty(world + 1, np.int32)
    rc = load_library().sfm_pcg_rank_rows(len(rp) - 1, ptr(rp), int(world), ptr(out))
    if rc != SFM_OK:
        raise ValueError(f"sfm_pcg_rank_rows failed ({rc})")
    return out


def device_count() -> int:
    """CUDA devices visible to the library (sfm_device_count)."""
    n = ctypes.c_int32()
    load_library().sfm_device_count(ctypes.byref(n))
    return n.value


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    rc = lib.sfm_nccl_unique_id(buf)
    if rc != SFM_OK:
        raise RuntimeError(f"ncclGetUniqueId failed ({rc})")
    return buf.raw


_default = {}
_default_lock = threading.Lock()


def default_context() -> Context:
    """Per-process context, created lazily: SFM_B200_DEVICES="0,1,..,7"
    makes it a single-process multi-GPU context (Context.multi), so the
    sfmkit-signature entry points (bundle_adjust, iterative_map) shard over
    those GPUs with no code change; otherwise cuda:SFM_B200_DEVICE /
    LOCAL_RANK / 0."""
    devs = os.environ.get("SFM_B200_DEVICES")
    if devs:
        key = "multi:" + devs
        with _default_lock:
            ctx = _default.get(key)
            if ctx is None:
                ctx = Context.multi([int(d) for d in devs.split(",") if d.strip()])
                _default[key] = ctx
            return ctx
    dev = int(os.environ.get("SFM_B200_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    with _default_lock:
        ctx = _default.get(dev)
        if ctx is None:
            ctx = Context(device=dev)
            _default[dev] = ctx
        return ctx


def set_default_context(ctx: Context):
    with _default_lock:
        _default[ctx.device] = ctx


def as_f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


def as_i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)
