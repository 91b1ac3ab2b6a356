"""cfg3 exploration (not a bench number): 1M-voxel scene, 800^2 training
step forward -> L1 -> backward, per-stage times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2412_04459_b200 as svr
from paper_2412_04459_b200.multiview import ShardedTrainer

ctx = svr.Context(0)
a = svr.synth_random_scene(7, 1 << 20, 9, 3)
scene = svr.Scene(ctx, a)
cam = svr.ring_camera(1, 0, 800, 800)
gt = np.random.default_rng(17).uniform(0, 1, (800, 800, 3))
tr = ShardedTrainer(ctx, scene, [cam], [gt], svr.RenderOptions(K=1, supersample=1.0, training=True))
for i in range(3):
    tr.step([0])
st = torch.cuda.ExternalStream(ctx.stream)
for rep in range(3):
    ctx.enable_timing(True)
    ctx.stage_times(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    loss = tr.step([0])
    e1.record(st)
    e1.synchronize()
    s = ctx.stage_times(reset=True)
    print(f"step {e0.elapsed_time(e1):.3f} ms loss {loss:.6f} contribs {tr.frame.info().n_contribs}",
          {k: round(x, 3) for k, x in s.items() if x > 0}, flush=True)
