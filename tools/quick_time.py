import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2412_04459_b200 as svr
ctx = svr.Context(0)
t=time.time(); a = svr.synth_random_scene(7, 1<<20, 9, 3); print("gen", time.time()-t, a.n_voxels, flush=True)
scene = svr.Scene(ctx, a)
cam = svr.ring_camera(1,0,1024,1024)
f = svr.Frame(ctx)
opts = svr.RenderOptions(supersample=1.0)
for i in range(3): svr.render_into(f, scene, cam, opts)
ctx.synchronize()
st = torch.cuda.ExternalStream(ctx.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
n=20
for i in range(n): svr.render_into(f, scene, cam, opts)
e1.record(st); e1.synchronize()
ms = e0.elapsed_time(e1)/n
inf = f.info()
print("ms/frame", ms, "FPS", 1000/ms, "E", inf.n_entries, "vis", inf.n_visible, "passes", inf.sort_passes, flush=True)
