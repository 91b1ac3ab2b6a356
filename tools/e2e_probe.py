import sys, time, torch
sys.path.insert(0, '.')
import paper_2412_04459_b200 as svr
ctx = svr.Context(0)
a = svr.synth_random_scene(7, 1 << 20, 9, 3)
scene = svr.Scene(ctx, a)
cam = svr.ring_camera(1, 0, 1024, 1024)
opts = svr.RenderOptions(supersample=1.0)
H = W = 1024
names = [("COLOR", 3), ("DEPTH", 1), ("MEDIAN_DEPTH", 1), ("NORMAL", 3), ("TRANSMITTANCE", 1)]
pinned = [{k: torch.empty(H * W * c, dtype=torch.float32, pin_memory=True) for k, c in names} for _ in range(2)]
frames = [svr.Frame(ctx), svr.Frame(ctx)]
def run(n, dl, mode):
    t_render = t_dl = t_wait = 0.0
    t0 = time.perf_counter()
    for i in range(n):
        f, host = frames[i % 2], pinned[i % 2]
        a0 = time.perf_counter(); f.wait(); a1 = time.perf_counter()
        svr.render_into(f, scene, cam, opts); a2 = time.perf_counter()
        if dl:
            for k, buf in host.items():
                if mode == "async": f.download_async(k, buf)
                else: f.download(k) if False else svr._check(svr.load_library().svr_frame_download(f.h, svr.BUF[k], svr.C.c_void_p(buf.data_ptr()), svr.C.c_size_t(buf.numel()*4)))
        a3 = time.perf_counter()
        t_wait += a1 - a0; t_render += a2 - a1; t_dl += a3 - a2
    for f in frames: f.wait()
    ctx.synchronize()
    tot = time.perf_counter() - t0
    print(f"{mode:6} dl={dl}: {1e3*tot/n:.3f} ms/step  host wait {1e3*t_wait/n:.3f} render {1e3*t_render/n:.3f} dl {1e3*t_dl/n:.3f}", flush=True)
for rep in range(2):
    run(50, False, "none"); run(50, True, "async"); run(50, True, "sync")
