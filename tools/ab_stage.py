"""Per-stage device time (CUDA events on the library stream) of a workload,
for A/B runs of build/env variants on the GPU box (never a bench number):
    python tools/ab_stage.py cfg2|cfg4|cfg3|cfg5 [frames]
(cfg5: one 1024^2 training view of the cfg4 scene per frame)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2412_04459_b200 as svr  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ctx = svr.Context(0)
if wl in ("cfg4", "cfg5"):
    a = svr.synth_unbounded_scene([svr.ring_camera(8, i, 1024, 1024) for i in range(8)], 7, 5, 2.8, seed=7)
    cams = [svr.ring_camera(256, v, 1024, 1024, 1.0) for v in range(int(os.environ.get("AB_VIEWS", "4")))]
else:
    a = svr.synth_random_scene(7, 1 << 20, 9, 3)
    res = 800 if wl == "cfg3" else 1024
    cams = [svr.ring_camera(256, v, res, res, 1.3) for v in range(8)]
scene = svr.Scene(ctx, a)
f = svr.Frame(ctx)
train = wl in ("cfg3", "cfg5")
opts = svr.RenderOptions(supersample=1.0, training=train)
if train:
    import torch
    R = cams[0].height
    gt = torch.rand(R, R, 3, device="cuda")
    gd = torch.zeros(a.n_pool, device="cuda")
    gs = torch.zeros(a.n_voxels * a.sh_stride, device="cuda")
    gp = torch.zeros(a.n_voxels, device="cuda")
    loss = torch.zeros(1, device="cuda")
    import ctypes as C
    g = svr.svr_gradients()
    g.density, g.sh, g.priority, g.on_device = gd.data_ptr(), gs.data_ptr(), gp.data_ptr(), 1
    lib = svr.load_library()

    def step(c):
        cc, oo = c.to_c(), opts.to_c()
        svr._check(lib.svr_train_step_l1(ctx.h, scene.h, C.byref(cc), C.byref(oo), gt.data_ptr(), f.h,
                                         C.byref(g), 0, loss.data_ptr()))
else:
    def step(c):
        svr.render_into(f, scene, c, opts)
for c in cams:
    step(c)
ctx.synchronize()
if os.environ.get("AB_ASYNC") == "1" and not train:  # deferred-E frames, as bench.py's render loop
    ctx.set_async(True)
    for c in cams:
        step(c)
        f.info()
    ctx.synchronize()
ctx.enable_timing(True)
ctx.stage_times(reset=True)
t = time.time()
for i in range(n):
    step(cams[i % len(cams)])
ctx.synchronize()
st = ctx.stage_times(reset=True)
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SVR_"))
print(wl, tag or "default", {k: round(v / n * 1000, 1) for k, v in st.items() if v > 0},
      "total_us", round(sum(st.values()) / n * 1000, 1), "E", f.info().n_entries, flush=True)
