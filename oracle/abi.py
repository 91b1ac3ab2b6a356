"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

The C structs of include/svr_b200.h (svr_camera, svr_render_options,
svr_scene_desc) and light value types for the CPU checkers, so that the
oracle front ends (oracle/ref.py, oracle/port.py) and bench.py's reference
arm never import the product package (and therefore never map
libsvr_b200.so). Every function here accepts the product's own Camera /
RenderOptions / SceneArrays objects too: they are read by attribute.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np


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


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    """std::invalid_argument in the reference."""


class LengthError(OracleError, OverflowError):
    """std::length_error in the reference."""


EXC = {1: InvalidArgument, 2: LengthError, 3: OracleError}


@dataclass
class Camera:
    """svr::Camera (camera.hpp:13-49)."""
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    rot: np.ndarray = field(default_factory=lambda: np.eye(3))
    pos: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def to_c(self) -> svr_camera:
        return camera_c(self)

    @staticmethod
    def from_c(c: svr_camera) -> "Camera":
        return Camera(c.width, c.height, c.fx, c.fy, c.cx, c.cy,
                      np.array(list(c.rot), dtype=np.float64).reshape(3, 3),
                      np.array(list(c.pos), dtype=np.float64))


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
        return options_c(self)


@dataclass
class SceneArrays:
    """svr::SparseScene (scene.hpp:21-46) as host arrays (same fields as the
    product's SceneArrays, so either can be handed to either side)."""
    codes: np.ndarray
    levels: np.ndarray
    corner_index: np.ndarray
    density: np.ndarray
    sh: np.ndarray
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


def camera_c(cam) -> svr_camera:
    """svr_camera of any camera-like object (ours or the product's)."""
    c = svr_camera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    r = np.asarray(cam.rot, dtype=np.float64).reshape(9)
    p = np.asarray(cam.pos, dtype=np.float64).reshape(3)
    for i in range(9):
        c.rot[i] = float(r[i])
    for i in range(3):
        c.pos[i] = float(p[i])
    return c


def options_c(o) -> svr_render_options:
    s = svr_render_options()
    s.K = int(o.K)
    s.t_threshold = float(o.t_threshold)
    s.supersample = float(o.supersample)
    for i in range(3):
        s.background[i] = float(o.background[i])
    s.near_plane = float(o.near_plane)
    s.far_sentinel = float(o.far_sentinel)
    s.record_stats = int(bool(o.record_stats))
    s.training = int(bool(o.training))
    return s


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class SceneDesc:
    """svr_scene_desc over host copies of a scene-like object's arrays (the
    copies stay alive as long as this object)."""

    def __init__(self, a):
        self.keep = [np.ascontiguousarray(a.codes, np.uint64),
                     np.ascontiguousarray(a.levels, np.uint8),
                     np.ascontiguousarray(a.corner_index, np.uint32).reshape(-1),
                     np.ascontiguousarray(a.density, np.float32),
                     np.ascontiguousarray(a.sh, np.float32).reshape(-1)]
        d = svr_scene_desc()
        d.n_voxels, d.n_pool, d.sh_degree = a.n_voxels, a.n_pool, int(a.sh_degree)
        for i in range(3):
            d.bounds_center[i] = float(a.bounds_center[i])
        d.bounds_size = float(a.bounds_size)
        d.codes, d.levels, d.corner_index, d.density, d.sh = [_p(x) for x in self.keep]
        self.d = d
