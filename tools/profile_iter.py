"""A few cfg3i device training iterations (for ncu launch lists; not a bench number)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2412_04459_b200 as svr
from paper_2412_04459_b200.trainer import DeviceTrainer
ctx = svr.Context(0)
a = svr.synth_random_scene(7, 1 << 20, 9, 3)
scene = svr.Scene(ctx, a)
cam = svr.ring_camera(1, 0, 800, 800)
gt = torch.tensor(np.random.default_rng(17).uniform(0, 1, (800, 800, 3)), dtype=torch.float32, device="cuda")
tr = DeviceTrainer(svr, ctx, scene, svr.RenderOptions(K=1, supersample=1.0))
for i in range(int(os.environ.get("ITERS", "3"))):
    tr.step(cam, gt)
ctx.synchronize()
