"""Max depth / colour error against the reference over several cfg4 and cfg1 views."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2412_04459_b200 as svr
from oracle import ref
ref.load_ref()
ctx = svr.Context(0)
cams = [svr.ring_camera(8, i, 1024, 1024) for i in range(8)]
arrays = svr.synth_unbounded_scene(cams, 7, 5, 2.8, seed=7)
scene = svr.Scene(ctx, arrays); rscene = ref.RefScene.from_arrays(arrays)
worst = 0
for view in [5, 40, 77, 130, 201]:
    cam = svr.ring_camera(256, view, 64, 64, 1.0)
    opts = svr.RenderOptions(supersample=1.0)
    out = svr.render(scene, cam, opts); r = ref.ref_render(rscene, cam, opts)
    m = r["depth"] < 1e20
    dd = np.abs(out.depth.astype(np.float64) - r["depth"])[m]
    print("cfg4 view", view, "depth max %.3e mean %.3e" % (dd.max(), dd.mean()), "color %.3e" % np.abs(out.color - r["color"]).max(),
          "median %.3e" % np.abs(out.median_depth.astype(np.float64) - r["median_depth"])[r["median_depth"] < 1e20].max() if hasattr(out, "median_depth") else "")
    worst = max(worst, dd.max())
a1 = svr.synth_random_scene(2024, 65536, 7, 3); s1 = svr.Scene(ctx, a1); r1 = ref.RefScene.generate(2024, 65536, 7, 3)
for K in [1, 2, 3]:
    cam = svr.ring_camera(1, 0, 256, 256)
    opts = svr.RenderOptions(K=K, supersample=1.0)
    out = svr.render(s1, cam, opts); r = ref.ref_render(r1, cam, opts)
    m = r["depth"] < 1e20
    print("cfg1 K", K, "depth max %.3e" % np.abs(out.depth.astype(np.float64) - r["depth"])[m].max(), "color %.3e" % np.abs(out.color - r["color"]).max())
print("worst cfg4 depth", worst)
