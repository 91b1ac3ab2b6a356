"""cfg4 exploration (not a bench number): 8M-voxel init_unbounded scene,
a few 1024^2 views from ring_cameras(256, ..., 1.0), per-stage times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_04459_b200 as svr

t = time.time()
cams8 = [svr.ring_camera(8, i, 1024, 1024) for i in range(8)]
a = svr.synth_unbounded_scene(cams8, 7, 5, 2.8, seed=7)
print("scene", a.n_voxels, a.n_pool, "gen s", round(time.time() - t, 1), flush=True)
ctx = svr.Context(0)
scene = svr.Scene(ctx, a)
f = svr.Frame(ctx)
opts = svr.RenderOptions(supersample=1.0)
views = [int(v) for v in os.environ.get("VIEWS", "0,1,77,128").split(",")]
for v in views:
    cam = svr.ring_camera(256, v, 1024, 1024, 1.0)
    for rep in range(3):
        ctx.enable_timing(True)
        ctx.stage_times(reset=True)
        t = time.time()
        svr.render_into(f, scene, cam, opts)
        ctx.synchronize()
        wall = time.time() - t
        st = ctx.stage_times(reset=True)
    inf = f.info()
    print(f"view {v}: E {inf.n_entries} vis {inf.n_visible} passes {inf.sort_passes} wall {wall*1e3:.2f} ms",
          {k: round(x, 3) for k, x in st.items() if x > 0}, flush=True)
    if os.environ.get("CHECK"):
        img = f.download("TRANSMITTANCE") if hasattr(f, "download") else None
