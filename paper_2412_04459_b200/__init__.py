"""B200-native sparse-voxel rasterizer (SVRaster render + gradient path).

Python host mirror of the reference's C++ rasterizer API
(`proj/include/svr/raster.hpp:52-141`) over the C ABI in
`include/svr_b200.h`, implemented by `libsvr_b200.so` (hand-written sm_100a
CUDA kernels, built in-tree by `make -C paper_2412_04459_b200`).

There is no CPU fallback: if the shared library or a CUDA device is missing,
every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SVR_LIB", os.path.join(_HERE, "libsvr_b200.so"))

TILE_SIZE = 16
TILE_ID_BITS = 16
VOXEL_ID_BITS = 29
MAX_LEVEL = 16

# svr_status (include/svr_b200.h) -> Python exceptions mirroring the
# reference's exception types.
OK, ERR_INVALID_ARGUMENT, ERR_LENGTH, ERR_RUNTIME, ERR_CUDA, ERR_NO_DEVICE = range(6)


class SvrError(RuntimeError):
    pass


class InvalidArgument(SvrError, ValueError):
    """std::invalid_argument in the reference."""


class LengthError(SvrError, OverflowError):
    """std::length_error in the reference."""


class RuntimeErrorSvr(SvrError):
    """std::runtime_error in the reference."""


class CudaError(SvrError):
    pass


class NoDeviceError(CudaError):
    pass


_EXC = {ERR_INVALID_ARGUMENT: InvalidArgument, ERR_LENGTH: LengthError,
        ERR_RUNTIME: RuntimeErrorSvr, ERR_CUDA: CudaError, ERR_NO_DEVICE: NoDeviceError}


class svr_camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("rot", C.c_double * 9), ("pos", C.c_double * 3)]


class svr_render_options(C.Structure):
    _fields_ = [("K", C.c_int32), ("t_threshold", C.c_double), ("supersample", C.c_double),
                ("background", C.c_double * 3), ("near_plane", C.c_double),
                ("far_sentinel", C.c_double), ("record_stats", C.c_int32),
                ("training", C.c_int32)]


class svr_scene_desc(C.Structure):
    _fields_ = [("n_voxels", C.c_uint64), ("n_pool", C.c_uint64), ("sh_degree", C.c_int32),
                ("bounds_center", C.c_double * 3), ("bounds_size", C.c_double),
                ("codes", C.c_void_p), ("levels", C.c_void_p), ("corner_index", C.c_void_p),
                ("density", C.c_void_p), ("sh", C.c_void_p)]


class svr_frame_info(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("ss_width", C.c_int32),
                ("ss_height", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
                ("n_visible", C.c_uint64), ("n_entries", C.c_uint64),
                ("n_contribs", C.c_uint64), ("sort_passes", C.c_int32), ("training", C.c_int32),
                ("composite_path", C.c_int32), ("reserved", C.c_int32)]


class svr_upstream(C.Structure):
    _fields_ = [("d_color", C.c_void_p), ("d_depth", C.c_void_p), ("d_normal", C.c_void_p),
                ("d_tfin_ss", C.c_void_p), ("d_weight", C.c_void_p),
                ("d_voxel_color", C.c_void_p), ("n_d_weight", C.c_uint64),
                ("n_d_voxel_color", C.c_uint64), ("on_device", C.c_int32)]


class svr_ray_loss_weights(C.Structure):
    _fields_ = [("w_T", C.c_double), ("w_dist", C.c_double), ("w_R", C.c_double)]


class svr_ray_loss_values(C.Structure):
    _fields_ = [("l_T", C.c_double), ("l_dist", C.c_double), ("l_R", C.c_double)]


class svr_gradients(C.Structure):
    _fields_ = [("density", C.c_void_p), ("sh", C.c_void_p), ("priority", C.c_void_p),
                ("on_device", C.c_int32)]


# svr_buffer ids
BUF = dict(COLOR=0, DEPTH=1, MEDIAN_DEPTH=2, NORMAL=3, TRANSMITTANCE=4, MAX_BLEND=5,
           SS_COLOR=6, SS_DEPTH=7, SS_TFIN=8, SORT_KEYS=9, SORT_VALUES=10, TILE_RANGES=11,
           TILE_MASKS=12, VOXEL_RECTS=13, VOXEL_AABB=14, ENTRIES_KEYS=15, ENTRIES_VALUES=16,
           PIX_COUNT=17, PIX_BEGIN=18, VOXEL_COLOR=19, VOXEL_NORMAL=20, OUTPUTS=21)

# exported symbols of include/svr_b200.h (checked by the CPU test-suite)
EXPORTS = [
    "svr_last_error", "svr_abi_version", "svr_ctx_create", "svr_ctx_destroy", "svr_ctx_stream",
    "svr_ctx_synchronize", "svr_ctx_set_async", "svr_ctx_overflow_count", "svr_ctx_set_debug", "svr_scene_upload", "svr_scene_set_params",
    "svr_scene_destroy", "svr_scene_param_ptrs", "svr_scene_save_svrx", "svr_scene_load_svrx",
    "svr_scene_info", "svr_scene_download", "svr_scene_prune", "svr_scene_subdivide",
    "svr_scene_remap", "svr_frame_create", "svr_frame_destroy",
    "svr_render", "svr_frame_get_info", "svr_frame_download", "svr_frame_device_ptr",
    "svr_frame_download_async", "svr_frame_wait", "svr_frame_records", "svr_render_backward",
    "svr_l1_loss", "svr_train_step_l1", "svr_ray_losses", "svr_adam_step", "svr_image_losses",
    "svr_project_voxels", "svr_tile_sign_masks", "svr_build_sort_entries", "svr_sort_entries",
    "svr_synth_random_scene", "svr_ring_camera", "svr_free", "svr_launch_count",
    "svr_ctx_enable_timing", "svr_ctx_stage_times", "svr_frame_pre", "svr_render_oracle",
    "svr_synth_unbounded_scene", "svr_frame_loss_values", "svr_ctx_take_adam_nan",
    "svr_host_alloc", "svr_host_free", "svr_comm_unique_id", "svr_comm_create",
    "svr_comm_destroy", "svr_comm_register", "svr_comm_check", "svr_comm_allreduce_gradients",
    "svr_train_batch_l1",
]
STAGES = ["tile_setup", "preprocess", "scan", "duplicate", "sort", "ranges", "composite",
          "record", "downsample", "backward", "epilogue", "other"]

_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads libsvr_b200.so. Raises (no fallback) when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `make -C {_HERE}` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    P = C.c_void_p
    sig = {
        "svr_last_error": (C.c_char_p, []),
        "svr_abi_version": (C.c_int, []),
        "svr_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
        "svr_ctx_destroy": (C.c_int, [P]),
        "svr_ctx_stream": (P, [P]),
        "svr_ctx_synchronize": (C.c_int, [P]),
        "svr_ctx_set_debug": (C.c_int, [P, C.c_int]),
        "svr_ctx_set_async": (C.c_int, [P, C.c_int]),
        "svr_ctx_overflow_count": (C.c_int, [P, C.POINTER(C.c_uint32)]),
        "svr_scene_upload": (C.c_int, [P, C.POINTER(svr_scene_desc), C.POINTER(P)]),
        "svr_scene_set_params": (C.c_int, [P, P, P, P, C.c_int]),
        "svr_scene_destroy": (C.c_int, [P]),
        "svr_scene_save_svrx": (C.c_int, [P, P, C.c_char_p]),
        "svr_scene_load_svrx": (C.c_int, [P, C.c_char_p, C.POINTER(P)]),
        "svr_scene_info": (C.c_int, [P, C.POINTER(svr_scene_desc)]),
        "svr_scene_prune": (C.c_int, [P, P, P, C.c_uint64, C.c_double, C.c_int32, C.POINTER(P)]),
        "svr_scene_subdivide": (C.c_int, [P, P, P, C.c_uint64, C.POINTER(P)]),
        "svr_scene_remap": (C.c_int, [P, P, P]),
        "svr_scene_download": (C.c_int, [P, P, P, P, P, P, P]),
        "svr_scene_param_ptrs": (C.c_int, [P, C.POINTER(P), C.POINTER(P),
                                           C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "svr_frame_create": (C.c_int, [P, C.POINTER(P)]),
        "svr_frame_download_async": (C.c_int, [P, C.c_int, P, C.c_size_t]),
        "svr_image_losses": (C.c_int, [P, P, P, C.c_double, C.c_double, P, P, C.c_int32]),
        "svr_frame_loss_values": (C.c_int, [P, P]),
        "svr_ctx_take_adam_nan": (C.c_int, [P, P]),
        "svr_adam_step": (C.c_int, [P, P, P, P, P, C.c_uint64, C.c_int64, C.c_double, C.c_double,
                                    C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                    C.c_int32]),
        "svr_ray_losses": (C.c_int, [P, P, P, C.POINTER(svr_ray_loss_weights),
                                     C.POINTER(svr_ray_loss_values), P, P, P, C.c_int32]),
        "svr_frame_wait": (C.c_int, [P]),
        "svr_frame_destroy": (C.c_int, [P]),
        "svr_render": (C.c_int, [P, P, C.POINTER(svr_camera), C.POINTER(svr_render_options), P]),
        "svr_frame_get_info": (C.c_int, [P, C.POINTER(svr_frame_info)]),
        "svr_frame_download": (C.c_int, [P, C.c_int, P, C.c_size_t]),
        "svr_frame_device_ptr": (C.c_int, [P, C.c_int, C.POINTER(P), C.POINTER(C.c_size_t)]),
        "svr_frame_records": (C.c_int, [P, P, C.c_uint64, P, P, P, C.c_uint64]),
        "svr_render_backward": (C.c_int, [P, P, P, C.POINTER(svr_upstream),
                                          C.POINTER(svr_gradients)]),
        "svr_l1_loss": (C.c_int, [P, P, P, P, P]),
        "svr_train_step_l1": (C.c_int, [P, P, C.POINTER(svr_camera),
                                        C.POINTER(svr_render_options), P, P,
                                        C.POINTER(svr_gradients), C.c_int, P]),
        "svr_project_voxels": (C.c_int, [P, C.POINTER(svr_camera), C.c_uint64, P, P, C.c_double,
                                         P, P, P]),
        "svr_tile_sign_masks": (C.c_int, [P, C.POINTER(svr_camera), P, C.c_uint64]),
        "svr_build_sort_entries": (C.c_int, [P, C.POINTER(svr_camera), C.c_uint64, C.c_uint64,
                                             P, P, P, P, P, C.c_uint64,
                                             C.POINTER(C.c_uint64)]),
        "svr_sort_entries": (C.c_int, [P, C.c_uint64, P, P]),
        "svr_synth_random_scene": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                             C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                             C.POINTER(P), C.POINTER(P), C.POINTER(P),
                                             C.POINTER(P), C.POINTER(P)]),
        "svr_synth_unbounded_scene": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_double,
                                                C.c_uint64, C.c_int, C.POINTER(C.c_uint64),
                                                C.POINTER(C.c_uint64)] + [C.POINTER(P)] * 5
                                      + [P, C.POINTER(C.c_double)]),
        "svr_ring_camera": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                      C.c_double, C.POINTER(svr_camera)]),
        "svr_free": (None, [P]),
        "svr_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(P)]),
        "svr_host_free": (C.c_int, [P]),
        "svr_comm_unique_id": (C.c_int, [P]),
        "svr_comm_create": (C.c_int, [P, P, C.c_int, C.c_int, C.POINTER(P)]),
        "svr_comm_destroy": (C.c_int, [P]),
        "svr_comm_register": (C.c_int, [P, P, C.c_size_t]),
        "svr_comm_check": (C.c_int, [P]),
        "svr_comm_allreduce_gradients": (C.c_int, [P, C.POINTER(svr_gradients), C.c_uint64,
                                                   C.c_uint64, C.c_uint64]),
        "svr_train_batch_l1": (C.c_int, [P, P, C.POINTER(svr_camera), C.POINTER(P), C.c_int,
                                         C.POINTER(svr_render_options), P,
                                         C.POINTER(svr_gradients), P, P]),
        "svr_launch_count": (C.c_ulonglong, []),
        "svr_ctx_enable_timing": (C.c_int, [P, C.c_int]),
        "svr_ctx_stage_times": (C.c_int, [P, C.POINTER(C.c_double), C.c_int, C.c_int]),
        "svr_frame_pre": (C.c_int, [P, P, C.c_uint64]),
        "svr_render_oracle": (C.c_int, [P, P, C.POINTER(svr_camera),
                                        C.POINTER(svr_render_options), P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status: int) -> None:
    if status != OK:
        msg = load_library().svr_last_error().decode(errors="replace")
        raise _EXC.get(status, SvrError)(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- value types
@dataclass
class Camera:
    """svr::Camera (camera.hpp:13-49): pinhole, row-major c2w rotation."""
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    rot: np.ndarray = field(default_factory=lambda: np.eye(3))
    pos: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def to_c(self) -> svr_camera:
        c = svr_camera()
        c.width, c.height = int(self.width), int(self.height)
        c.fx, c.fy, c.cx, c.cy = float(self.fx), float(self.fy), float(self.cx), float(self.cy)
        r = np.asarray(self.rot, dtype=np.float64).reshape(9)
        p = np.asarray(self.pos, dtype=np.float64).reshape(3)
        for i in range(9):
            c.rot[i] = float(r[i])
        for i in range(3):
            c.pos[i] = float(p[i])
        return c

    @staticmethod
    def from_c(c: svr_camera) -> "Camera":
        return Camera(c.width, c.height, c.fx, c.fy, c.cx, c.cy,
                      np.array(list(c.rot), dtype=np.float64).reshape(3, 3),
                      np.array(list(c.pos), dtype=np.float64))


def ring_camera(n_views: int, index: int, width: int, height: int, distance: float = 1.3,
                fov_x_deg: float = 55.0) -> Camera:
    """ring_cameras (synth.cpp:89-118), camera `index` of `n_views`."""
    c = svr_camera()
    _check(load_library().svr_ring_camera(n_views, index, width, height, distance, fov_x_deg,
                                          C.byref(c)))
    return Camera.from_c(c)


@dataclass
class RenderOptions:
    """svr::RenderOptions (raster.hpp:22-31) with the reference's defaults."""
    K: int = 1
    t_threshold: float = 1e-4
    supersample: float = 1.5
    background: Sequence[float] = (0.0, 0.0, 0.0)
    near_plane: float = 1e-6
    far_sentinel: float = 1e30
    record_stats: bool = False
    training: bool = False

    def to_c(self) -> svr_render_options:
        o = svr_render_options()
        o.K = int(self.K)
        o.t_threshold = float(self.t_threshold)
        o.supersample = float(self.supersample)
        for i in range(3):
            o.background[i] = float(self.background[i])
        o.near_plane = float(self.near_plane)
        o.far_sentinel = float(self.far_sentinel)
        o.record_stats = int(bool(self.record_stats))
        o.training = int(bool(self.training))
        return o


@dataclass
class SceneArrays:
    """svr::SparseScene (scene.hpp:21-46) as host arrays."""
    codes: np.ndarray          # u64 [N]
    levels: np.ndarray         # u8  [N]
    corner_index: np.ndarray   # u32 [N, 8]
    density: np.ndarray        # f32 [P]
    sh: np.ndarray             # f32 [N, stride]
    sh_degree: int = 3
    bounds_center: Sequence[float] = (0.0, 0.0, 0.0)
    bounds_size: float = 1.0

    @property
    def n_voxels(self) -> int:
        return int(self.codes.shape[0])

    @property
    def n_pool(self) -> int:
        return int(self.density.shape[0])

    @property
    def sh_stride(self) -> int:
        return 3 * (self.sh_degree + 1) ** 2


def _take_scene(lib, n, p, ptrs, sh_degree, **kw) -> SceneArrays:
    N, P = n.value, p.value
    stride = 3 * (sh_degree + 1) ** 2

    def take(ptr, dtype, count):
        buf = (C.c_char * (max(count, 1) * np.dtype(dtype).itemsize)).from_address(ptr.value)
        arr = np.frombuffer(buf, dtype=dtype, count=count).copy()
        lib.svr_free(ptr)
        return arr

    return SceneArrays(take(ptrs[0], np.uint64, N), take(ptrs[1], np.uint8, N),
                       take(ptrs[2], np.uint32, N * 8).reshape(N, 8),
                       take(ptrs[3], np.float32, P), take(ptrs[4], np.float32, N * stride)
                       .reshape(N, stride), sh_degree, **kw)


def synth_random_scene(seed: int, target: int, max_level: int, sh_degree: int = 3) -> SceneArrays:
    """Generator G of SURVEY §8(d) (same RNG stream as the oracle's)."""
    lib = load_library()
    n, p = C.c_uint64(), C.c_uint64()
    ptrs = [C.c_void_p() for _ in range(5)]
    _check(lib.svr_synth_random_scene(seed, target, max_level, sh_degree, C.byref(n), C.byref(p),
                                      *[C.byref(x) for x in ptrs]))
    return _take_scene(lib, n, p, ptrs, sh_degree)


def synth_unbounded_scene(cameras: Sequence["Camera"], init_level: int = 7, shell_levels: int = 5,
                          bg_ratio: float = 2.8, seed: int = 7,
                          sh_degree: int = 3) -> SceneArrays:
    """init_unbounded (optim.cpp:96-184) over `cameras`, parameters randomised
    as generator G from mt19937_64(seed): the config-4/5 scene of SURVEY §8(d)
    is synth_unbounded_scene([ring_camera(8, i, 1024, 1024) for i in range(8)])."""
    lib = load_library()
    arr = (svr_camera * len(cameras))(*[c.to_c() for c in cameras])
    n, p = C.c_uint64(), C.c_uint64()
    ptrs = [C.c_void_p() for _ in range(5)]
    bc = (C.c_double * 3)()
    bs = C.c_double()
    _check(lib.svr_synth_unbounded_scene(arr, len(cameras), init_level, shell_levels, bg_ratio,
                                         seed, sh_degree, C.byref(n), C.byref(p),
                                         *[C.byref(x) for x in ptrs], bc, C.byref(bs)))
    return _take_scene(lib, n, p, ptrs, sh_degree, bounds_center=tuple(bc), bounds_size=bs.value)


# ---------------------------------------------------------------- handles
class Context:
    """One per (host thread, device): a CUDA stream plus scratch arenas."""

    def __init__(self, device: int = 0, debug: bool = False):
        self._lib = load_library()
        h = C.c_void_p()
        _check(self._lib.svr_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        if debug:
            _check(self._lib.svr_ctx_set_debug(h, 1))

    @property
    def stream(self) -> int:
        return int(self._lib.svr_ctx_stream(self.h) or 0)

    def synchronize(self) -> None:
        _check(self._lib.svr_ctx_synchronize(self.h))

    def set_async(self, on: bool = True) -> None:
        """Deferred-E rendering (svr_ctx_set_async)."""
        _check(self._lib.svr_ctx_set_async(self.h, int(on)))

    def overflow_count(self) -> int:
        n = C.c_uint32()
        _check(self._lib.svr_ctx_overflow_count(self.h, C.byref(n)))
        return int(n.value)

    def enable_timing(self, on: bool = True) -> None:
        _check(self._lib.svr_ctx_enable_timing(self.h, int(on)))

    def stage_times(self, reset: bool = True) -> dict:
        buf = (C.c_double * len(STAGES))()
        _check(self._lib.svr_ctx_stage_times(self.h, buf, len(STAGES), int(reset)))
        return {k: buf[i] for i, k in enumerate(STAGES)}

    def close(self) -> None:
        if getattr(self, "h", None):
            self._lib.svr_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def launch_count() -> int:
    """Kernels launched by libsvr_b200.so so far (process-wide)."""
    return int(load_library().svr_launch_count())


class Scene:
    """Device-resident SparseScene."""

    def __init__(self, ctx: Context, arrays: SceneArrays):
        self.ctx = ctx
        self.arrays = arrays
        a = arrays
        self._keep = [np.ascontiguousarray(a.codes, dtype=np.uint64),
                      np.ascontiguousarray(a.levels, dtype=np.uint8),
                      np.ascontiguousarray(a.corner_index, dtype=np.uint32).reshape(-1),
                      np.ascontiguousarray(a.density, dtype=np.float32),
                      np.ascontiguousarray(a.sh, dtype=np.float32).reshape(-1)]
        d = svr_scene_desc()
        d.n_voxels, d.n_pool, d.sh_degree = a.n_voxels, a.n_pool, int(a.sh_degree)
        for i in range(3):
            d.bounds_center[i] = float(a.bounds_center[i])
        d.bounds_size = float(a.bounds_size)
        d.codes, d.levels, d.corner_index, d.density, d.sh = [_ptr(x) for x in self._keep]
        h = C.c_void_p()
        _check(ctx._lib.svr_scene_upload(ctx.h, C.byref(d), C.byref(h)))
        self.h = h
        self._keep = None

    @property
    def n_voxels(self) -> int:
        return self.arrays.n_voxels

    @property
    def n_pool(self) -> int:
        return self.arrays.n_pool

    @classmethod
    def load_svrx(cls, ctx: Context, path: str) -> "Scene":
        """load_checkpoint (io.cpp:281-359) straight into a device scene
        (svr_scene_load_svrx); `arrays` is read back from the device."""
        h = C.c_void_p()
        _check(ctx._lib.svr_scene_load_svrx(ctx.h, os.fsencode(path), C.byref(h)))
        return cls._adopt(ctx, h)

    @classmethod
    def _adopt(cls, ctx: Context, h) -> "Scene":
        """Wraps a scene created on the device; its host `arrays` are read
        back on first use."""
        self = cls.__new__(cls)
        self.ctx, self.h, self._keep = ctx, h, None
        self._arrays = None
        return self

    @property
    def arrays(self) -> SceneArrays:
        if getattr(self, "_arrays", None) is None:
            self._arrays = self.download()
        return self._arrays

    @arrays.setter
    def arrays(self, value: SceneArrays) -> None:
        self._arrays = value

    def prune(self, max_blend_weight, threshold: float) -> "Scene":
        """prune (optim.cpp:207-234) on the device: a new scene."""
        st = np.ascontiguousarray(max_blend_weight, dtype=np.float32).reshape(-1)
        h = C.c_void_p()
        _check(self.ctx._lib.svr_scene_prune(self.ctx.h, self.h, _ptr(st), st.size, threshold, 0,
                                             C.byref(h)))
        return Scene._adopt(self.ctx, h)

    def subdivide(self, selected) -> "Scene":
        """subdivide_voxels (optim.cpp:236-298) on the device: a new scene."""
        sel = np.ascontiguousarray(selected, dtype=np.uint32).reshape(-1)
        h = C.c_void_p()
        _check(self.ctx._lib.svr_scene_subdivide(self.ctx.h, self.h, _ptr(sel), sel.size,
                                                 C.byref(h)))
        return Scene._adopt(self.ctx, h)

    def remap(self):
        """AdaptRemap of an adapted scene: (voxel_src, pool_src), -1 = new."""
        vs = np.empty(self.arrays.n_voxels, np.int64)
        ps = np.empty(self.arrays.n_pool, np.int64)
        _check(self.ctx._lib.svr_scene_remap(self.h, _ptr(vs), _ptr(ps)))
        return vs, ps

    def save_svrx(self, path: str) -> None:
        """save_checkpoint (io.cpp:250-279) of the scene's current device parameters."""
        _check(self.ctx._lib.svr_scene_save_svrx(self.ctx.h, self.h, os.fsencode(path)))

    def download(self) -> SceneArrays:
        """The device scene as host arrays (svr_scene_info + svr_scene_download)."""
        d = svr_scene_desc()
        _check(self.ctx._lib.svr_scene_info(self.h, C.byref(d)))
        n, p, deg = int(d.n_voxels), int(d.n_pool), int(d.sh_degree)
        stride = 3 * (deg + 1) ** 2
        codes = np.empty(n, np.uint64)
        levels = np.empty(n, np.uint8)
        ci = np.empty((n, 8), np.uint32)
        dens = np.empty(p, np.float32)
        sh = np.empty((n, stride), np.float32)
        _check(self.ctx._lib.svr_scene_download(self.ctx.h, self.h, _ptr(codes), _ptr(levels),
                                                _ptr(ci), _ptr(dens), _ptr(sh)))
        return SceneArrays(codes, levels, ci, dens, sh, deg, tuple(d.bounds_center),
                           float(d.bounds_size))

    def set_params(self, density=None, sh=None, on_device: bool = False) -> None:
        """PoolsD refresh (raster.hpp:47-52). Host numpy arrays or device pointers."""
        if on_device:
            _check(self.ctx._lib.svr_scene_set_params(self.ctx.h, self.h, density, sh, 1))
            return
        d = None if density is None else np.ascontiguousarray(density, dtype=np.float32)
        s = None if sh is None else np.ascontiguousarray(sh, dtype=np.float32)
        _check(self.ctx._lib.svr_scene_set_params(self.ctx.h, self.h, _ptr(d), _ptr(s), 0))

    def param_ptrs(self):
        d, s = C.c_void_p(), C.c_void_p()
        npool, nsh = C.c_uint64(), C.c_uint64()
        _check(self.ctx._lib.svr_scene_param_ptrs(self.h, C.byref(d), C.byref(s), C.byref(npool),
                                                  C.byref(nsh)))
        return d.value, s.value, npool.value, nsh.value

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx._lib.svr_scene_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Frame:
    """Per-view device state; the device half of svr::ForwardRecords."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        h = C.c_void_p()
        _check(ctx._lib.svr_frame_create(ctx.h, C.byref(h)))
        self.h = h

    def info(self) -> svr_frame_info:
        i = svr_frame_info()
        _check(self.ctx._lib.svr_frame_get_info(self.h, C.byref(i)))
        return i

    def device_ptr(self, which: str):
        p, n = C.c_void_p(), C.c_size_t()
        _check(self.ctx._lib.svr_frame_device_ptr(self.h, BUF[which], C.byref(p), C.byref(n)))
        return p.value, n.value

    def download(self, which: str, dtype, shape=None) -> np.ndarray:
        _, nbytes = self.device_ptr(which)
        out = np.empty(nbytes // np.dtype(dtype).itemsize, dtype=dtype)
        _check(self.ctx._lib.svr_frame_download(self.h, BUF[which], _ptr(out), C.c_size_t(nbytes)))
        return out if shape is None else out.reshape(shape)

    def download_async(self, which: str, out) -> None:
        """Enqueues the read-back of buffer `which` into `out` (a contiguous
        numpy array or CPU tensor of the buffer's size, pinned for overlap);
        `out` is complete after wait()."""
        ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        nbytes = out.numel() * out.element_size() if hasattr(out, "numel") else out.nbytes
        _check(self.ctx._lib.svr_frame_download_async(self.h, BUF[which], C.c_void_p(ptr),
                                                      C.c_size_t(nbytes)))

    def wait(self) -> None:
        """Blocks until this frame's asynchronous downloads have landed."""
        _check(self.ctx._lib.svr_frame_wait(self.h))

    def records(self):
        """(pre_vids, contrib_pre, contrib_a, contrib_b, pix_begin, pix_count)."""
        inf = self.info()
        pre = np.empty(inf.n_visible, dtype=np.uint32)
        cp = np.empty(inf.n_contribs, dtype=np.uint32)
        ca = np.empty(inf.n_contribs, dtype=np.float64)
        cb = np.empty(inf.n_contribs, dtype=np.float64)
        _check(self.ctx._lib.svr_frame_records(self.h, _ptr(pre), inf.n_visible, _ptr(cp), _ptr(ca),
                                               _ptr(cb), inf.n_contribs))
        pb = self.download("PIX_BEGIN", np.uint32)
        pc = self.download("PIX_COUNT", np.uint32)
        return pre, cp, ca, cb, pb, pc

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx._lib.svr_frame_destroy(self.h)
                self.h = None
        except Exception:
            pass


@dataclass
class RenderOutput:
    """svr::RenderOutput (raster.hpp:84-92), float32 images."""
    color: np.ndarray
    depth: np.ndarray
    median_depth: np.ndarray
    normal: np.ndarray
    transmittance: np.ndarray
    max_blend_weight: Optional[np.ndarray]
    frame: Frame


@dataclass
class SceneGradients:
    """svr::SceneGradients (raster.hpp:94-98), float32."""
    density: np.ndarray
    sh: np.ndarray
    priority: np.ndarray


def render_into(frame: Frame, scene: Scene, cam: Camera, opts: RenderOptions) -> None:
    """Device-only render (no download)."""
    c, o = cam.to_c(), opts.to_c()
    _check(scene.ctx._lib.svr_render(scene.ctx.h, scene.h, C.byref(c), C.byref(o), frame.h))


def render(scene: Scene, cam: Camera, opts: RenderOptions = RenderOptions(),
           frame: Optional[Frame] = None) -> RenderOutput:
    """svr::render / render_with_pools (raster.cpp:205-301) on the GPU."""
    f = frame or Frame(scene.ctx)
    render_into(f, scene, cam, opts)
    H, W = cam.height, cam.width
    mb = f.download("MAX_BLEND", np.float32) if opts.record_stats else None
    return RenderOutput(f.download("COLOR", np.float32, (H, W, 3)),
                        f.download("DEPTH", np.float32, (H, W)),
                        f.download("MEDIAN_DEPTH", np.float32, (H, W)),
                        f.download("NORMAL", np.float32, (H, W, 3)),
                        f.download("TRANSMITTANCE", np.float32, (H, W)), mb, f)


def render_backward(scene: Scene, frame: Frame, d_color=None, d_depth=None, d_normal=None,
                    d_tfin_ss=None, d_weight=None, d_voxel_color=None) -> SceneGradients:
    """svr::render_backward (raster.cpp:303-423); host upstream -> host gradients."""
    keep = [None if x is None else np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
            for x in (d_color, d_depth, d_normal, d_tfin_ss, d_weight, d_voxel_color)]
    u = svr_upstream()
    u.d_color, u.d_depth, u.d_normal, u.d_tfin_ss, u.d_weight, u.d_voxel_color = \
        [_ptr(x) for x in keep]
    u.n_d_weight = 0 if keep[4] is None else keep[4].size
    u.n_d_voxel_color = 0 if keep[5] is None else keep[5].size // 3
    u.on_device = 0
    a = scene.arrays
    gd = np.empty(a.n_pool, np.float32)
    gs = np.empty(a.n_voxels * a.sh_stride, np.float32)
    gp = np.empty(a.n_voxels, np.float32)
    g = svr_gradients()
    g.density, g.sh, g.priority, g.on_device = _ptr(gd), _ptr(gs), _ptr(gp), 0
    _check(scene.ctx._lib.svr_render_backward(scene.ctx.h, scene.h, frame.h, C.byref(u),
                                              C.byref(g)))
    return SceneGradients(gd, gs.reshape(a.n_voxels, a.sh_stride), gp)


def ray_losses(frame: Frame, gt, w_T: float = 0.0, w_dist: float = 0.0, w_R: float = 0.0,
               d_tfin_ss=None, d_weight=None, d_voxel_color=None):
    """svr::ray_losses (losses.cpp:141-238) on the device over `frame`'s
    forward records. Host path: the gradient arrays (float32, created zeroed
    when None) are accumulated into and returned with the loss values:
    ((l_T, l_dist, l_R), d_tfin_ss, d_weight, d_voxel_color)."""
    inf = frame.info()
    nss, nc = inf.ss_width * inf.ss_height, inf.n_contribs
    g = np.ascontiguousarray(gt, dtype=np.float32).reshape(-1)
    dtf = np.zeros(nss, np.float32) if d_tfin_ss is None else d_tfin_ss
    dw = np.zeros(nc, np.float32) if d_weight is None else d_weight
    dvc = np.zeros(nc * 3, np.float32) if d_voxel_color is None else d_voxel_color
    w = svr_ray_loss_weights(w_T, w_dist, w_R)
    v = svr_ray_loss_values()
    _check(frame.ctx._lib.svr_ray_losses(frame.ctx.h, frame.h, _ptr(g), C.byref(w), C.byref(v),
                                         _ptr(dtf), _ptr(dw), _ptr(dvc), 0))
    return (v.l_T, v.l_dist, v.l_R), dtf, dw, dvc.reshape(-1, 3)


def image_losses(frame: Frame, gt, w_mse: float = 1.0, w_ssim: float = 0.0, d_color=None):
    """mse_loss + ssim_loss (losses.cpp:71-139) of the frame's colour vs gt on
    the device: ((mse, 1 - ssim), d_color), d_color (float32 W*H*3, created
    zeroed when None) accumulated with w_mse*dMSE + w_ssim*d(1-SSIM)."""
    g = np.ascontiguousarray(gt, dtype=np.float32).reshape(-1)
    d = np.zeros(g.size, np.float32) if d_color is None else d_color
    out = (C.c_double * 2)()
    _check(frame.ctx._lib.svr_image_losses(frame.ctx.h, frame.h, _ptr(g), w_mse, w_ssim, out,
                                           _ptr(d), 0))
    return (out[0], out[1]), d.reshape(gt.shape)


class AdamState:
    """optim.hpp:112-115 on the device: fp64 moments, step count."""

    def __init__(self, n: int, device: int = 0):
        import torch
        dev = torch.device("cuda", device)
        self.m = torch.zeros(n, dtype=torch.float64, device=dev)
        self.v = torch.zeros(n, dtype=torch.float64, device=dev)
        self.step = 0


def adam_step(ctx: Context, params, grads, state: AdamState, lr: float, lr_alt: float = 0.0,
              period: int = 0, n_primary: int = 0, beta1: float = 0.1, beta2: float = 0.99,
              eps: float = 1e-15) -> None:
    """svr::adam_step (optim.cpp:322-345) on device tensors (float32 params
    and grads, the AdamState's fp64 moments), in place on the context stream."""
    state.step += 1
    _check(ctx._lib.svr_adam_step(ctx.h, C.c_void_p(params.data_ptr()),
                                  C.c_void_p(grads.data_ptr()), C.c_void_p(state.m.data_ptr()),
                                  C.c_void_p(state.v.data_ptr()), params.numel(), state.step, lr,
                                  lr_alt, period, n_primary, beta1, beta2, eps, 1))


# ---------------------------------------------------------------- pipeline pieces
def project_voxels(ctx: Context, cam: Camera, centers: np.ndarray, sizes: np.ndarray,
                   near_plane: float = 1e-6):
    """project_voxel (raster.cpp:72-118) for a batch; returns (visible, aabb, rect)."""
    centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1, 3)
    sizes = np.ascontiguousarray(sizes, dtype=np.float64).reshape(-1)
    n = sizes.size
    vis = np.empty(n, np.uint8)
    aabb = np.empty((n, 4), np.float64)
    rect = np.empty((n, 4), np.int32)
    c = cam.to_c()
    _check(ctx._lib.svr_project_voxels(ctx.h, C.byref(c), n, _ptr(centers), _ptr(sizes),
                                       near_plane, _ptr(vis), _ptr(aabb), _ptr(rect)))
    return vis.astype(bool), aabb, rect


def tile_sign_masks(ctx: Context, cam: Camera) -> np.ndarray:
    """tile_sign_patterns (raster.cpp:120-142) for all tiles, as bitmasks."""
    ntx = (cam.width + 15) // 16
    nty = (cam.height + 15) // 16
    out = np.empty(ntx * nty, np.uint8)
    c = cam.to_c()
    _check(ctx._lib.svr_tile_sign_masks(ctx.h, C.byref(c), _ptr(out), out.size))
    return out


def tile_sign_patterns(ctx: Context, cam: Camera, tx: int, ty: int) -> list:
    m = int(tile_sign_masks(ctx, cam)[ty * ((cam.width + 15) // 16) + tx])
    return [s for s in range(8) if m >> s & 1]


def build_sort_entries(ctx: Context, cam: Camera, scene_voxel_count: int, vids: np.ndarray,
                       codes: np.ndarray, rects: np.ndarray):
    """build_sort_entries (raster.cpp:144-172); returns (keys u64, values u32)."""
    vids = np.ascontiguousarray(vids, dtype=np.uint32)
    codes = np.ascontiguousarray(codes, dtype=np.uint64)
    rects = np.ascontiguousarray(rects, dtype=np.int32).reshape(-1, 4)
    c = cam.to_c()
    n = C.c_uint64()
    _check(ctx._lib.svr_build_sort_entries(ctx.h, C.byref(c), scene_voxel_count, vids.size,
                                           _ptr(vids), _ptr(codes), _ptr(rects), None, None, 0,
                                           C.byref(n)))
    keys = np.empty(n.value, np.uint64)
    vals = np.empty(n.value, np.uint32)
    _check(ctx._lib.svr_build_sort_entries(ctx.h, C.byref(c), scene_voxel_count, vids.size,
                                           _ptr(vids), _ptr(codes), _ptr(rects), _ptr(keys),
                                           _ptr(vals), n.value, C.byref(n)))
    return keys, vals


def sort_entries(ctx: Context, keys: np.ndarray, values: np.ndarray):
    """sort_entries (raster.cpp:174-178): ascending (key, value) on the GPU."""
    k = np.ascontiguousarray(keys, dtype=np.uint64).copy()
    v = np.ascontiguousarray(values, dtype=np.uint32).copy()
    _check(ctx._lib.svr_sort_entries(ctx.h, k.size, _ptr(k), _ptr(v)))
    return k, v
