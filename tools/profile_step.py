"""A few cfg2 renders for ncu (never a bench number)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_04459_b200 as svr
ctx = svr.Context(0)
a = svr.synth_random_scene(7, 1 << 20, 9, 3)
scene = svr.Scene(ctx, a)
f = svr.Frame(ctx)
opts = svr.RenderOptions(supersample=float(os.environ.get("SVR_SS", "1.0")))
for i in range(int(os.environ.get("SVR_FRAMES", "3"))):
    svr.render_into(f, scene, svr.ring_camera(1, 0, 1024, 1024), opts)
ctx.synchronize()
print("frames done, launches:", svr.launch_count())
