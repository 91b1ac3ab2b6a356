"""Tile entry-count distribution of view 0 of the cfg2 and cfg4 workloads (the
measurement behind DESIGN §8's per-tile composite-path note; GPU box):
    python tools/tile_lengths.py"""
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2412_04459_b200 as svr
ctx = svr.Context(0)
for wl in ("cfg2", "cfg4"):
    if wl == "cfg4":
        a = svr.synth_unbounded_scene([svr.ring_camera(8, i, 1024, 1024) for i in range(8)], 7, 5, 2.8, seed=7)
        cam = svr.ring_camera(256, 0, 1024, 1024, 1.0)
    else:
        a = svr.synth_random_scene(7, 1 << 20, 9, 3)
        cam = svr.ring_camera(256, 0, 1024, 1024, 1.3)
    sc = svr.Scene(ctx, a); f = svr.Frame(ctx)
    svr.render_into(f, sc, cam, svr.RenderOptions(supersample=1.0))
    r = f.download("TILE_RANGES", np.uint32, (-1, 2)).astype(np.int64)
    L = np.maximum(r[:, 1] - r[:, 0], 0)
    E = L.sum()
    for t in (512, 1024, 2048, 4096, 8192):
        m = L >= t
        print(wl, "tiles>=%d: %d of %d, entries share %.3f" % (t, m.sum(), L.size, L[m].sum() / E))
    print(wl, "max", L.max(), "mean", L.mean())
