"""One iteration of the reference training loop on the device.

optim::train (optim.cpp:433-495) runs, per iteration: render (training) ->
mse_loss + lambda_ssim * ssim_loss -> ray_losses (lambda_T, lambda_dist,
lambda_R) -> render_backward -> priority += -> adam_step on the density pool
and on the SH pool (band 0 at lr_sh0, the rest at lr_sh_rest). DeviceTrainer
chains the C-ABI entry points that implement those steps (svr_render,
svr_image_losses, svr_ray_losses, svr_render_backward, svr_adam_step) with
every buffer resident on the GPU; the scene's own parameter pools are updated
in place. Adaptation (prune / subdivide), the TV loss (lambda_tv = 1e-10 in
the defaults) and the mesh-mode normal-depth losses are not part of it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np


@dataclass
class TrainWeights:
    """The TrainConfig fields one iteration uses (optim.hpp:39-60 defaults)."""
    lr_density: float = 0.025
    lr_sh0: float = 0.01
    lr_sh_rest: float = 0.00025
    adam_beta1: float = 0.1
    adam_beta2: float = 0.99
    adam_eps: float = 1e-15
    lambda_ssim: float = 0.02
    lambda_T: float = 0.01
    lambda_dist: float = 0.1   # the reference applies it from iteration dist_from on
    lambda_R: float = 0.01


class DeviceTrainer:
    def __init__(self, svr, ctx, scene, opts, weights: TrainWeights = TrainWeights()):
        import torch
        self.svr, self.ctx, self.scene, self.w = svr, ctx, scene, weights
        self.opts = opts
        self.opts.training = True
        self.dev = torch.device("cuda", ctx.device)
        self.frame = svr.Frame(ctx)
        d_ptr, s_ptr, n_pool, n_sh = scene.param_ptrs()
        self.d_ptr, self.s_ptr, self.n_pool, self.n_sh = d_ptr, s_ptr, n_pool, n_sh
        a = scene.arrays
        self.stride = a.sh_stride
        f32, f64 = torch.float32, torch.float64
        self.g_density = torch.zeros(n_pool, dtype=f32, device=self.dev)
        self.g_sh = torch.zeros(n_sh, dtype=f32, device=self.dev)
        self.g_priority = torch.zeros(a.n_voxels, dtype=f32, device=self.dev)
        self.priority = torch.zeros(a.n_voxels, dtype=f32, device=self.dev)  # optim.cpp:477
        self.m_d = torch.zeros(n_pool, dtype=f64, device=self.dev)
        self.v_d = torch.zeros(n_pool, dtype=f64, device=self.dev)
        self.m_s = torch.zeros(n_sh, dtype=f64, device=self.dev)
        self.v_s = torch.zeros(n_sh, dtype=f64, device=self.dev)
        self.step_count = 0
        self._bufs = {}

    def _buf(self, name, n):
        import torch
        b = self._bufs.get(name)
        if b is None or b.numel() < n:
            b = torch.empty(max(n, 1), dtype=torch.float32, device=self.dev)
            self._bufs[name] = b
        return b[:max(n, 1)]

    def gradients(self, cam, gt_device, with_dist: bool = True, defer: bool = False) -> dict:
        """Forward + all losses + backward; fills g_density / g_sh / g_priority.
        Returns the loss values (TrainLogEntry fields); with defer the losses
        stay on the device (read them with loss_values()) and nothing waits."""
        svr, lib, ctx, f = self.svr, self.ctx._lib, self.ctx, self.frame
        svr.render_into(f, self.scene, cam, self.opts)
        inf = f.info()
        W, H = cam.width, cam.height
        nss, nc = inf.ss_width * inf.ss_height, inf.n_contribs
        d_color = self._buf("d_color", W * H * 3)
        d_tfin = self._buf("d_tfin", nss)
        d_weight = self._buf("d_weight", nc)
        d_vc = self._buf("d_vc", nc * 3)
        with self._on_stream():  # cleared on the library stream: no host wait
            for b in (d_color, d_tfin, d_weight, d_vc):
                b.zero_()
        mode = 2 if defer else 1
        img = (C.c_double * 2)()
        svr._check(lib.svr_image_losses(ctx.h, f.h, C.c_void_p(gt_device.data_ptr()), 1.0,
                                        self.w.lambda_ssim, img, C.c_void_p(d_color.data_ptr()), mode))
        rw = svr.svr_ray_loss_weights(self.w.lambda_T, self.w.lambda_dist if with_dist else 0.0,
                                      self.w.lambda_R)
        rv = svr.svr_ray_loss_values()
        svr._check(lib.svr_ray_losses(ctx.h, f.h, C.c_void_p(gt_device.data_ptr()), C.byref(rw),
                                      C.byref(rv), C.c_void_p(d_tfin.data_ptr()),
                                      C.c_void_p(d_weight.data_ptr()), C.c_void_p(d_vc.data_ptr()),
                                      mode))
        u = svr.svr_upstream()
        u.d_color, u.d_tfin_ss = d_color.data_ptr(), d_tfin.data_ptr()
        u.d_weight, u.d_voxel_color = d_weight.data_ptr(), d_vc.data_ptr()
        u.n_d_weight, u.n_d_voxel_color, u.on_device = nc, nc, 1
        g = svr.svr_gradients()
        g.density, g.sh, g.priority = (self.g_density.data_ptr(), self.g_sh.data_ptr(),
                                       self.g_priority.data_ptr())
        g.on_device = 1
        svr._check(lib.svr_render_backward(ctx.h, self.scene.h, f.h, C.byref(u), C.byref(g)))
        if defer:
            return {}
        return {"l_mse": img[0], "l_ssim": img[1], "l_T": rv.l_T, "l_dist": rv.l_dist,
                "l_R": rv.l_R}

    def loss_values(self) -> dict:
        """The frame's last loss values (one host wait)."""
        out = (C.c_double * 5)()
        self.svr._check(self.ctx._lib.svr_frame_loss_values(self.frame.h, out))
        return {"l_mse": out[0], "l_ssim": out[1], "l_T": out[2], "l_dist": out[3], "l_R": out[4]}

    def step(self, cam, gt_device, with_dist: bool = True, lr_decay: float = 1.0) -> dict:
        """One training iteration (optim.cpp:433-495 minus adaptation). The
        whole iteration is enqueued without a host wait; the loss values and
        Adam's NaN check are read once at the end."""
        svr, lib, ctx, w = self.svr, self.ctx._lib, self.ctx, self.w
        self.gradients(cam, gt_device, with_dist, defer=True)
        with self._on_stream():
            self.priority += self.g_priority
        self.step_count += 1
        svr._check(lib.svr_adam_step(ctx.h, C.c_void_p(self.d_ptr),
                                     C.c_void_p(self.g_density.data_ptr()),
                                     C.c_void_p(self.m_d.data_ptr()), C.c_void_p(self.v_d.data_ptr()),
                                     self.n_pool, self.step_count, w.lr_density * lr_decay, 0.0, 0, 0,
                                     w.adam_beta1, w.adam_beta2, w.adam_eps, 2))
        svr._check(lib.svr_adam_step(ctx.h, C.c_void_p(self.s_ptr), C.c_void_p(self.g_sh.data_ptr()),
                                     C.c_void_p(self.m_s.data_ptr()), C.c_void_p(self.v_s.data_ptr()),
                                     self.n_sh, self.step_count, w.lr_sh0 * lr_decay,
                                     w.lr_sh_rest * lr_decay, self.stride, 3, w.adam_beta1,
                                     w.adam_beta2, w.adam_eps, 2))
        log = self.loss_values()
        nan = C.c_int32()
        svr._check(lib.svr_ctx_take_adam_nan(ctx.h, C.byref(nan)))
        if nan.value:
            raise RuntimeError("adam_step: NaN gradient")  # optim.cpp:337-338 (std::runtime_error)
        rw_dist = w.lambda_dist if with_dist else 0.0
        log["total"] = (log["l_mse"] + w.lambda_ssim * log["l_ssim"] + w.lambda_T * log["l_T"] +
                        rw_dist * log["l_dist"] + w.lambda_R * log["l_R"])
        return log

    def _on_stream(self):
        import torch
        return torch.cuda.stream(torch.cuda.ExternalStream(self.ctx.stream, device=self.dev))

    def params(self):
        """Host copies of the (device-updated) density and SH pools."""
        self.ctx.synchronize()
        return [device_to_host(ptr, n) for ptr, n in ((self.d_ptr, self.n_pool),
                                                      (self.s_ptr, self.n_sh))]


class _DevArray:
    """A raw float32 device pointer as a __cuda_array_interface__ object."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3}


def device_to_host(ptr: int, n: int) -> np.ndarray:
    import torch
    return torch.as_tensor(_DevArray(ptr, n), device="cuda").cpu().numpy()
