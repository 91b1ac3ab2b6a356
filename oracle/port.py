"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes front end of oracle/_ref/libsvr_oracle.so, the plain-C restatement
(svr_oracle.c) of the reference render and gradient path. Builds it with gcc
on first use when the prebuilt .so is absent (gcc is in the image).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from oracle import abi
from oracle.abi import camera_c, options_c

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_ref", "libsvr_oracle.so")
_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO):
        subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
    lib = C.CDLL(SO)
    P = C.c_void_p
    desc = C.POINTER(abi.svr_scene_desc)
    cam = C.POINTER(abi.svr_camera)
    opt = C.POINTER(abi.svr_render_options)
    for name, args in {
        "orc_tile_masks": [cam, P],
        "orc_project": [desc, cam, C.c_double, P, P, P],
        "orc_entries": [desc, cam, C.c_double, C.c_int, C.POINTER(C.c_uint64), P, P],
        "orc_render": [desc, cam, opt, P, P, P, P, P, P],
        "orc_backward": [desc, cam, opt, P, P, P, P, P, P, P],
    }.items():
        fn = getattr(lib, name)
        fn.restype = C.c_int
        fn.argtypes = args
    _lib = lib
    return lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _Desc(abi.SceneDesc):
    pass


def _chk(st):
    if st != 0:
        raise abi.EXC.get(st, abi.OracleError)(f"oracle status {st}")


def tile_masks(cam):
    out = np.empty(((cam.width + 15) // 16) * ((cam.height + 15) // 16), np.uint8)
    c = camera_c(cam)
    _chk(load().orc_tile_masks(C.byref(c), _p(out)))
    return out


def project(a, cam, near=1e-6):
    d = _Desc(a)
    n = a.n_voxels
    vis, aabb, rect = np.empty(n, np.uint8), np.empty((n, 4)), np.empty((n, 4), np.int32)
    c = camera_c(cam)
    _chk(load().orc_project(C.byref(d.d), C.byref(c), near, _p(vis), _p(aabb), _p(rect)))
    return vis.astype(bool), aabb, rect


def entries(a, cam, sorted_, near=1e-6):
    d = _Desc(a)
    c = camera_c(cam)
    n = C.c_uint64()
    _chk(load().orc_entries(C.byref(d.d), C.byref(c), near, int(sorted_), C.byref(n), None, None))
    k, v = np.empty(n.value, np.uint64), np.empty(n.value, np.uint32)
    _chk(load().orc_entries(C.byref(d.d), C.byref(c), near, int(sorted_), C.byref(n), _p(k), _p(v)))
    return k, v


def render(a, cam, opts):
    d = _Desc(a)
    W, H = cam.width, cam.height
    out = {"color": np.empty((H, W, 3)), "depth": np.empty((H, W)), "median_depth": np.empty((H, W)),
           "normal": np.empty((H, W, 3)), "transmittance": np.empty((H, W))}
    mb = np.empty(a.n_voxels) if opts.record_stats else None
    c, o = camera_c(cam), options_c(opts)
    _chk(load().orc_render(C.byref(d.d), C.byref(c), C.byref(o), _p(out["color"]), _p(out["depth"]),
                           _p(out["median_depth"]), _p(out["normal"]), _p(out["transmittance"]), _p(mb)))
    out["max_blend_weight"] = mb
    return out


def backward(a, cam, opts, d_color=None, d_depth=None, d_normal=None, d_tfin_ss=None):
    d = _Desc(a)
    keep = [None if x is None else np.ascontiguousarray(x, np.float64)
            for x in (d_color, d_depth, d_normal, d_tfin_ss)]
    gd, gs, gp = np.empty(a.n_pool), np.empty(a.n_voxels * a.sh_stride), np.empty(a.n_voxels)
    c, o = camera_c(cam), options_c(opts)
    _chk(load().orc_backward(C.byref(d.d), C.byref(c), C.byref(o), *[_p(x) for x in keep],
                             _p(gd), _p(gs), _p(gp)))
    return {"density": gd, "sh": gs.reshape(a.n_voxels, a.sh_stride), "priority": gp}
