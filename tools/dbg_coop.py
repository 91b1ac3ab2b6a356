"""Debug: one training render of config 3 (scene G 1M, 800^2) and config 2 render images vs the non-coop kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_04459_b200 as svr
ctx = svr.Context(0)
a = svr.synth_random_scene(7, 1 << 20, 9, 3)
scene = svr.Scene(ctx, a)
res = int(os.environ.get("RES", "800"))
cam = svr.ring_camera(256, 0, res, res, 1.3)
train = os.environ.get("TRAIN", "1") == "1"
out = svr.render(scene, cam, svr.RenderOptions(supersample=1.0, training=train))
print("ok", out.frame.info().n_contribs, float(out.color.mean()), flush=True)
