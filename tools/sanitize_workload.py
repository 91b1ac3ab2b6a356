"""Small end-to-end workload for compute-sanitizer (tests/test_gpu_sanitizer.py):
forward (K 1-3, supersampled, stats, training records on both composite
paths), backward with every upstream kind, ray/image losses, Adam, and the
deferred-E path including a frame that outgrows its entry capacity."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2412_04459_b200 as svr  # noqa: E402

ctx = svr.Context(0)
a = svr.synth_random_scene(2024, 6000, 6, 3)
scene = svr.Scene(ctx, a)
cam = svr.ring_camera(1, 0, 48, 40)
for K, ss, stats in [(1, 1.0, False), (2, 1.5, True), (3, 1.0, False)]:
    out = svr.render(scene, cam, svr.RenderOptions(K=K, supersample=ss, record_stats=stats,
                                                   background=(0.1, 0.2, 0.3)))
opts = svr.RenderOptions(K=2, supersample=1.5, training=True)
out = svr.render(scene, cam, opts)
inf = out.frame.info()
rng = np.random.default_rng(0)
gt = rng.uniform(0, 1, (40, 48, 3)).astype(np.float32)
(lt, ld, lr), dtf, dw, dvc = svr.ray_losses(out.frame, gt, 0.01, 0.1, 0.01)
(lm, ls), dcol = svr.image_losses(out.frame, gt, 1.0, 0.02)
g = svr.render_backward(scene, out.frame, d_color=dcol, d_depth=rng.uniform(-1, 1, (40, 48)),
                        d_normal=rng.uniform(-1, 1, (40, 48, 3)), d_tfin_ss=dtf, d_weight=dw,
                        d_voxel_color=dvc)
assert np.isfinite(g.density).all() and np.isfinite(g.sh).all()
# deferred entry count: a frame sized on a small scene, then an outgrowing one
actx = svr.Context(0)
actx.set_async(True)
small = svr.Scene(actx, svr.synth_random_scene(3, 600, 5, 3))
big = svr.Scene(actx, a)
f = svr.Frame(actx)
svr.render_into(f, small, cam, svr.RenderOptions(supersample=1.0))
for sc in (small, big, big):
    svr.render_into(f, sc, cam, svr.RenderOptions(supersample=1.0))
    f.download("COLOR", np.float32)
print("sanitize workload ok", inf.n_entries, inf.n_contribs, actx.overflow_count())
