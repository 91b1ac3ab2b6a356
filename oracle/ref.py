"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes front end of the CPU checkers:
  * `oracle/_ref/libsvr_ref.so`: the UNMODIFIED reference C++ sources
    (/root/reference/proj/src/{scene,image,raster,losses,synth}.cpp) behind
    the extern "C" shim `oracle/ref_shim.cpp` (built by `make -C oracle ref`).
  * `oracle/_ref/libsvr_oracle.so`: the plain-C restatement `svr_oracle.c`
    (built by `make -C oracle oracle`), pinned against the former.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsvr_ref.so")
PORT_SO = os.path.join(HERE, "_ref", "libsvr_oracle.so")

_ref = None
_port = None


from oracle import abi
from oracle.abi import camera_c, options_c


def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir("/root/reference/proj")


def load_ref() -> C.CDLL:
    global _ref
    if _ref is not None:
        return _ref
    if not os.path.exists(REF_SO):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-C", HERE, "ref"], check=True, capture_output=True)
        else:
            raise FileNotFoundError(f"{REF_SO} missing and /root/reference absent")
    lib = C.CDLL(REF_SO)
    P = C.c_void_p
    cam = C.POINTER(abi.svr_camera)
    opt = C.POINTER(abi.svr_render_options)
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_scene_gen": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.POINTER(P)]),
        "ref_scene_unbounded": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                          C.c_int, C.POINTER(P)]),
        "ref_scene_bounds": (None, [P, P, C.POINTER(C.c_double)]),
        "ref_scene_make": (C.c_int, [C.POINTER(abi.svr_scene_desc), C.POINTER(P)]),
        "ref_scene_from_paths": (C.c_int, [P, P, C.c_uint64, C.c_float, C.c_int, C.POINTER(P)]),
        "ref_scene_free": (None, [P]),
        "ref_scene_sizes": (None, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_int)]),
        "ref_scene_export": (None, [P, P, P, P, P, P]),
        "ref_scene_set_params": (None, [P, P, P]),
        "ref_ring_camera": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                      cam]),
        "ref_scaled_camera": (C.c_int, [cam, C.c_double, cam]),
        "ref_render": (C.c_int, [P, cam, opt, C.c_int, P, P, P, P, P, P]),
        "ref_project": (C.c_int, [P, cam, C.c_double, P, P, P]),
        "ref_project_one": (C.c_int, [cam, P, C.c_double, C.c_double, P, P, C.POINTER(C.c_int)]),
        "ref_tile_masks": (C.c_int, [cam, P]),
        "ref_entries": (C.c_int, [P, cam, C.c_double, C.c_int, C.POINTER(C.c_uint64), P, P]),
        "ref_sort_entries": (C.c_int, [C.c_uint64, P, P]),
        "ref_forward_train": (C.c_int, [P, cam, opt, C.POINTER(P), C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64), P, P, P, P]),
        "ref_frame_free": (None, [P]),
        "ref_frame_records": (None, [P, P, P, P, P, P, P, P]),
        "ref_backward": (C.c_int, [P, P, P, P, P, P, P, C.c_uint64, P, C.c_uint64, P, P, P]),
        "ref_train_step_l1": (C.c_int, [P, cam, opt, P, C.POINTER(C.c_double), P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _ref = lib
    return lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _chk(st):
    if st != 0:
        msg = load_ref().ref_last_error().decode()
        raise abi.EXC.get(st, abi.OracleError)(msg)


class RefScene:
    """A reference svr::SparseScene living in the oracle library."""

    def __init__(self, handle):
        self.h = handle

    @staticmethod
    def generate(seed: int, target: int, max_level: int, sh_degree: int = 3) -> "RefScene":
        h = C.c_void_p()
        _chk(load_ref().ref_scene_gen(seed, target, max_level, sh_degree, C.byref(h)))
        return RefScene(h)

    @staticmethod
    def unbounded(cameras, init_level: int, shell_levels: int, bg_ratio: float, seed: int,
                  sh_degree: int = 3) -> "RefScene":
        """init_unbounded (optim.cpp:96-184) + G-style parameters."""
        arr = (abi.svr_camera * len(cameras))(*[camera_c(c) for c in cameras])
        h = C.c_void_p()
        _chk(load_ref().ref_scene_unbounded(arr, len(cameras), init_level, shell_levels,
                                            bg_ratio, seed, sh_degree, C.byref(h)))
        return RefScene(h)

    def bounds(self):
        c = (C.c_double * 3)()
        s = C.c_double()
        load_ref().ref_scene_bounds(self.h, c, C.byref(s))
        return tuple(c), s.value

    @staticmethod
    def from_arrays(a) -> "RefScene":
        d = abi.SceneDesc(a)
        h = C.c_void_p()
        _chk(load_ref().ref_scene_make(C.byref(d.d), C.byref(h)))
        return RefScene(h)

    @staticmethod
    def from_paths(codes, levels, fill: float, sh_degree: int) -> "RefScene":
        codes = np.ascontiguousarray(codes, np.uint64)
        levels = np.ascontiguousarray(levels, np.uint8)
        h = C.c_void_p()
        _chk(load_ref().ref_scene_from_paths(_p(codes), _p(levels), codes.size, fill, sh_degree,
                                             C.byref(h)))
        return RefScene(h)

    def sizes(self):
        """(n_voxels, n_pool, sh_degree) without exporting the arrays."""
        n, p, deg = C.c_uint64(), C.c_uint64(), C.c_int()
        load_ref().ref_scene_sizes(self.h, C.byref(n), C.byref(p), C.byref(deg))
        return n.value, p.value, deg.value

    def arrays(self):
        n, p, deg = C.c_uint64(), C.c_uint64(), C.c_int()
        lib = load_ref()
        lib.ref_scene_sizes(self.h, C.byref(n), C.byref(p), C.byref(deg))
        N, P, D = n.value, p.value, deg.value
        stride = 3 * (D + 1) ** 2
        codes = np.empty(N, np.uint64)
        levels = np.empty(N, np.uint8)
        ci = np.empty((N, 8), np.uint32)
        dens = np.empty(P, np.float32)
        sh = np.empty((N, stride), np.float32)
        lib.ref_scene_export(self.h, _p(codes), _p(levels), _p(ci), _p(dens), _p(sh))
        c, s = self.bounds()
        return abi.SceneArrays(codes, levels, ci, dens, sh, D, c, s)

    def save_checkpoint(self, path: str) -> None:
        """save_checkpoint (io.cpp:250-279), the reference's SVRX writer."""
        lib = load_ref()
        lib.ref_save_checkpoint.argtypes = [C.c_void_p, C.c_char_p]
        _chk(lib.ref_save_checkpoint(self.h, os.fsencode(path)))

    @staticmethod
    def load_checkpoint(path: str) -> "RefScene":
        """load_checkpoint (io.cpp:283-359), the reference's SVRX reader."""
        lib = load_ref()
        lib.ref_load_checkpoint.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        h = C.c_void_p()
        _chk(lib.ref_load_checkpoint(os.fsencode(path), C.byref(h)))
        return RefScene(h)

    def set_params(self, density=None, sh=None):
        d = None if density is None else np.ascontiguousarray(density, np.float32)
        s = None if sh is None else np.ascontiguousarray(sh, np.float32)
        load_ref().ref_scene_set_params(self.h, _p(d), _p(s))

    def __del__(self):
        try:
            if self.h:
                load_ref().ref_scene_free(self.h)
        except Exception:
            pass


def ref_ring_camera(n, i, w, h, dist=1.3, fov=55.0):
    c = abi.svr_camera()
    _chk(load_ref().ref_ring_camera(n, i, w, h, dist, fov, C.byref(c)))
    return abi.Camera.from_c(c)


def ref_scaled_camera(cam, ss):
    c, o = camera_c(cam), abi.svr_camera()
    _chk(load_ref().ref_scaled_camera(C.byref(c), ss, C.byref(o)))
    return abi.Camera.from_c(o)


def ref_render(scene: RefScene, cam, opts, oracle: bool = False, n_voxels: int = 0):
    """svr::render (or render_oracle): dict of double images at target res."""
    W, H = cam.width, cam.height
    out = {"color": np.empty((H, W, 3)), "depth": np.empty((H, W)),
           "median_depth": np.empty((H, W)), "normal": np.empty((H, W, 3)),
           "transmittance": np.empty((H, W))}
    mb = np.empty(n_voxels) if opts.record_stats else None
    c, o = camera_c(cam), options_c(opts)
    _chk(load_ref().ref_render(scene.h, C.byref(c), C.byref(o), int(oracle), _p(out["color"]),
                               _p(out["depth"]), _p(out["median_depth"]), _p(out["normal"]),
                               _p(out["transmittance"]), _p(mb)))
    out["max_blend_weight"] = mb
    return out


def ref_project(scene: RefScene, cam, n_voxels: int, near: float = 1e-6):
    vis = np.empty(n_voxels, np.uint8)
    aabb = np.empty((n_voxels, 4))
    rect = np.empty((n_voxels, 4), np.int32)
    c = camera_c(cam)
    _chk(load_ref().ref_project(scene.h, C.byref(c), near, _p(vis), _p(aabb), _p(rect)))
    return vis.astype(bool), aabb, rect


def ref_tile_masks(cam):
    ntx, nty = (cam.width + 15) // 16, (cam.height + 15) // 16
    out = np.empty(ntx * nty, np.uint8)
    c = camera_c(cam)
    _chk(load_ref().ref_tile_masks(C.byref(c), _p(out)))
    return out


def ref_entries(scene: RefScene, cam, sorted_: bool, near: float = 1e-6):
    lib = load_ref()
    c = camera_c(cam)
    n = C.c_uint64()
    _chk(lib.ref_entries(scene.h, C.byref(c), near, int(sorted_), C.byref(n), None, None))
    keys = np.empty(n.value, np.uint64)
    vals = np.empty(n.value, np.uint32)
    _chk(lib.ref_entries(scene.h, C.byref(c), near, int(sorted_), C.byref(n), _p(keys), _p(vals)))
    return keys, vals


def ref_entries_both(scene: RefScene, cam, near: float = 1e-6):
    """(emitted keys, values, sorted keys, values) of one view, the entry
    list built once (build_sort_entries, then sort_entries on the same list)."""
    lib = load_ref()
    lib.ref_entries_begin.argtypes = [C.c_void_p, C.POINTER(abi.svr_camera), C.c_double,
                                      C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]
    lib.ref_entries_copy.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    lib.ref_entries_end.argtypes = [C.c_void_p]
    lib.ref_entries_end.restype = None
    c = camera_c(cam)
    h, n = C.c_void_p(), C.c_uint64()
    _chk(lib.ref_entries_begin(scene.h, C.byref(c), near, C.byref(h), C.byref(n)))
    try:
        out = []
        for sort_first in (0, 1):
            k, v = np.empty(n.value, np.uint64), np.empty(n.value, np.uint32)
            _chk(lib.ref_entries_copy(h, sort_first, _p(k), _p(v)))
            out += [k, v]
    finally:
        lib.ref_entries_end(h)
    return tuple(out)


def ref_sort_entries(keys, vals):
    k = np.ascontiguousarray(keys, np.uint64).copy()
    v = np.ascontiguousarray(vals, np.uint32).copy()
    _chk(load_ref().ref_sort_entries(k.size, _p(k), _p(v)))
    return k, v


class RefFrame:
    def __init__(self, scene: RefScene, cam, opts):
        self.scene = scene
        lib = load_ref()
        W, H = cam.width, cam.height
        self.color = np.empty((H, W, 3))
        self.depth = np.empty((H, W))
        self.normal = np.empty((H, W, 3))
        self.transmittance = np.empty((H, W))
        h = C.c_void_p()
        npre, nc = C.c_uint64(), C.c_uint64()
        c, o = camera_c(cam), options_c(opts)
        _chk(lib.ref_forward_train(scene.h, C.byref(c), C.byref(o), C.byref(h), C.byref(npre),
                                   C.byref(nc), _p(self.color), _p(self.depth), _p(self.normal),
                                   _p(self.transmittance)))
        self.h = h
        self.n_pre, self.n_contribs = npre.value, nc.value
        ss = ref_scaled_camera(cam, opts.supersample)
        self.sw, self.sh = ss.width, ss.height

    def records(self):
        pre = np.empty(self.n_pre, np.uint32)
        cp = np.empty(self.n_contribs, np.uint32)
        ca = np.empty(self.n_contribs)
        cb = np.empty(self.n_contribs)
        pb = np.empty(self.sw * self.sh, np.uint32)
        pc = np.empty(self.sw * self.sh, np.uint32)
        tf = np.empty(self.sw * self.sh)
        load_ref().ref_frame_records(self.h, _p(pre), _p(cp), _p(ca), _p(cb), _p(pb), _p(pc), _p(tf))
        return pre, cp, ca, cb, pb, pc, tf

    def ray_losses(self, gt, w_T=0.0, w_dist=0.0, w_R=0.0):
        """svr::ray_losses (losses.cpp:141-238) on this frame's records:
        ((l_T, l_dist, l_R), d_tfin_ss, d_weight, d_voxel_color)."""
        g = np.ascontiguousarray(gt, np.float64).reshape(-1)
        vals = np.zeros(3)
        dtf = np.zeros(self.sw * self.sh)
        dw = np.zeros(self.n_contribs)
        dvc = np.zeros(self.n_contribs * 3)
        _chk(load_ref().ref_frame_ray_losses(self.h, _p(g), C.c_double(w_T), C.c_double(w_dist),
                                             C.c_double(w_R), _p(vals), _p(dtf), _p(dw), _p(dvc)))
        return tuple(vals), dtf, dw, dvc.reshape(-1, 3)

    def backward(self, n_pool, n_sh, n_vox, d_color=None, d_depth=None, d_normal=None,
                 d_tfin_ss=None, d_weight=None, d_voxel_color=None):
        keep = [None if x is None else np.ascontiguousarray(x, np.float64).reshape(-1)
                for x in (d_color, d_depth, d_normal, d_tfin_ss, d_weight, d_voxel_color)]
        gd, gs, gp = np.empty(n_pool), np.empty(n_sh), np.empty(n_vox)
        nw = 0 if keep[4] is None else keep[4].size
        nvc = 0 if keep[5] is None else keep[5].size // 3
        _chk(load_ref().ref_backward(self.scene.h, self.h, _p(keep[0]), _p(keep[1]), _p(keep[2]),
                                     _p(keep[3]), _p(keep[4]), nw, _p(keep[5]), nvc, _p(gd),
                                     _p(gs), _p(gp)))
        return gd, gs, gp

    def __del__(self):
        try:
            load_ref().ref_frame_free(self.h)
        except Exception:
            pass


def ref_train_iteration_grads(scene: RefScene, cam, opts, gt, lambda_ssim, w_T, w_dist, w_R,
                              n_pool, n_sh, n_vox):
    """Loss values (mse, 1-ssim, l_T, l_dist, l_R) and the SceneGradients of one
    optim::train iteration (optim.cpp:433-477), before the Adam updates."""
    g = np.ascontiguousarray(gt, np.float64)
    losses = np.zeros(5)
    gd, gs, gp = np.empty(n_pool), np.empty(n_sh), np.empty(n_vox)
    c, o = camera_c(cam), options_c(opts)
    _chk(load_ref().ref_train_iteration_grads(scene.h, C.byref(c), C.byref(o), _p(g),
                                              C.c_double(lambda_ssim), C.c_double(w_T),
                                              C.c_double(w_dist), C.c_double(w_R), _p(losses),
                                              _p(gd), _p(gs), _p(gp)))
    return losses, gd, gs, gp


def ref_adapt(scene: RefScene, prune_stats=None, threshold=0.0, selected=None):
    """prune (stats, threshold) or subdivide_voxels (selected) of the
    reference (optim.cpp:207-298): (new RefScene, voxel_src, pool_src)."""
    n = scene.arrays().n_voxels
    lib = load_ref()
    h = C.c_void_p()
    nv, npool = C.c_uint64(), C.c_uint64()
    if prune_stats is not None:
        st = np.ascontiguousarray(prune_stats, np.float64)
        vs, ps = np.empty(max(n, 1), np.int64), np.empty(max(8 * n, 1), np.int64)
        _chk(lib.ref_prune(scene.h, _p(st), C.c_double(threshold), C.byref(h), _p(vs), _p(ps),
                           C.byref(nv), C.byref(npool)))
    else:
        sel = np.ascontiguousarray(selected, np.uint32)
        cap = n + 7 * sel.size
        vs, ps = np.empty(max(cap, 1), np.int64), np.empty(max(8 * cap, 1), np.int64)
        _chk(lib.ref_subdivide(scene.h, _p(sel), C.c_uint64(sel.size), C.byref(h), _p(vs), _p(ps),
                               C.byref(nv), C.byref(npool)))
    return RefScene(h), vs[:nv.value].copy(), ps[:npool.value].copy()


def ref_image_losses(a, b, w_mse, w_ssim, grads=True):
    """mse_loss + ssim_loss (losses.cpp:71-139): ((mse, 1 - ssim), d)."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    H, W = a.shape[:2]
    out = np.zeros(2)
    d = np.zeros_like(a) if grads else None
    _chk(load_ref().ref_image_losses(_p(a), _p(b), W, H, C.c_double(w_mse), C.c_double(w_ssim),
                                     _p(out), _p(d)))
    return tuple(out), d


def ref_adam_step(params, grads, m, v, step_before, lr, lr_alt=0.0, period=0, n_primary=0,
                  beta1=0.1, beta2=0.99, eps=1e-15):
    """svr::adam_step (optim.cpp:322-345) on copies; returns (params, m, v)."""
    p = np.ascontiguousarray(params, np.float32).copy()
    g = np.ascontiguousarray(grads, np.float64)
    mm = np.ascontiguousarray(m, np.float64).copy()
    vv = np.ascontiguousarray(v, np.float64).copy()
    _chk(load_ref().ref_adam_step(_p(p), _p(g), _p(mm), _p(vv), C.c_uint64(p.size),
                                  C.c_int64(step_before), C.c_double(lr), C.c_double(lr_alt),
                                  C.c_uint32(period), C.c_uint32(n_primary), C.c_double(beta1),
                                  C.c_double(beta2), C.c_double(eps)))
    return p, mm, vv


def ref_train_step_l1(scene: RefScene, cam, opts, gt, n_pool, n_sh, n_vox):
    c, o = camera_c(cam), options_c(opts)
    gt = np.ascontiguousarray(gt, np.float64)
    loss = C.c_double()
    dcol = np.empty_like(gt)
    gd, gs, gp = np.empty(n_pool), np.empty(n_sh), np.empty(n_vox)
    _chk(load_ref().ref_train_step_l1(scene.h, C.byref(c), C.byref(o), _p(gt), C.byref(loss),
                                      _p(dcol), _p(gd), _p(gs), _p(gp)))
    return loss.value, dcol, gd, gs, gp
