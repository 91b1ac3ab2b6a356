"""Timing of device adaptation on the config-2 scene vs the reference (not a bench line)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_04459_b200 as svr
from oracle import ref
ref.load_ref()
ctx = svr.Context(0)
a = svr.synth_random_scene(7, 1 << 20, 9, 3)
scene = svr.Scene(ctx, a)
rscene = ref.RefScene.from_arrays(a)
rng = np.random.default_rng(3)
stats = rng.uniform(0, 1, a.n_voxels).astype(np.float32)
sel = rng.choice(a.n_voxels, a.n_voxels // 20, replace=False).astype(np.uint32)  # subdiv_percent 5
for name, fn, rfn in [("prune(thr 0.05)", lambda: scene.prune(stats, 0.05),
                       lambda: ref.ref_adapt(rscene, prune_stats=stats.astype(np.float64), threshold=0.05)),
                      ("subdivide(5%)", lambda: scene.subdivide(sel), lambda: ref.ref_adapt(rscene, selected=sel))]:
    fn(); ctx.synchronize()
    t = time.perf_counter(); s2 = fn(); ctx.synchronize(); dt = time.perf_counter() - t
    t = time.perf_counter(); rfn(); rdt = time.perf_counter() - t
    print(f"{name}: device {dt*1e3:.1f} ms (device scene incl. its rank table), "
          f"reference {rdt*1e3:.0f} ms (1 core); new voxels {s2.arrays.n_voxels} pool {s2.arrays.n_pool}", flush=True)
