"""Per-stage device time of config-2 frames (CUDA events on the library stream)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_04459_b200 as svr
ctx = svr.Context(0)
a = svr.synth_random_scene(7, 1 << 20, 9, 3)
scene = svr.Scene(ctx, a)
f = svr.Frame(ctx)
opts = svr.RenderOptions(supersample=1.0)
cams = [svr.ring_camera(256, v, 1024, 1024, 1.3) for v in range(8)]
for c in cams: svr.render_into(f, scene, c, opts)
ctx.synchronize()
ctx.enable_timing(True); ctx.stage_times(reset=True)
n = 40
for i in range(n): svr.render_into(f, scene, cams[i % 8], opts)
ctx.synchronize()
st = ctx.stage_times(reset=True)
print(os.environ.get("SVR_RANK_ORDER", "1"), {k: round(v / n * 1000, 1) for k, v in st.items() if v > 0}, "total us", round(sum(st.values()) / n * 1000, 1))
